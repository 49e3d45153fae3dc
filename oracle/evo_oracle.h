/* evo_oracle.h — CPU restatement of the reference's Evoformer attention path.
 *
 * TEST INFRASTRUCTURE ONLY. This is the parity checker for the CUDA kernels
 * in paper_2310_04610_b200/csrc; only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it. The product path never calls it.
 *
 * Semantics follow /root/reference/proj/core/src/attention_tiled.cpp
 * (attn_forward_tiled :57-180, attn_backward_tiled :182-340) operation for
 * operation, including the per-op rounding of the problem format
 * (numeric_format.hpp:64-65: F32 rounds through (float), F64 is exact).
 * Extension not present in the reference (parity of this part is pinned
 * only by finite differences and by bias1 == 0 bit-identity): a per-row key
 * mask bias1[b, j] (DeepSpeed's [Bo, N, 1, 1, L]) added after the scaled
 * dot product and before the pair bias, and an outer batch Bo for the pair
 * bias bias2[Bo, H, L, L] (the reference's (H, L, L) bias is Bo == 1).
 *
 * Layouts (row-major, canonical axes of attention.hpp:24-31):
 *   q, k, v, o, do, dq, dk, dv : (B, L, H, D)   with B = Bo * N
 *   bias1, dbias1              : (B, L)
 *   bias2, dbias2              : (Bo, H, L, L)
 *   lse                        : (H, B, L)     natural-log units
 * All arrays are double; values are exactly representable in `fmt`.
 */
#ifndef EVO_ORACLE_H
#define EVO_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { EVO_ORACLE_F64 = 0, EVO_ORACLE_F32 = 1 };

typedef struct {
  int fmt;          /* EVO_ORACLE_F64 / EVO_ORACLE_F32 */
  int64_t B, L, H, D;
  int64_t Bo;       /* outer batch of bias2; B % Bo == 0 */
  double scale;
  int64_t tile_q, tile_k, tile_b; /* attention_tiled.hpp:15-18 */
  int deterministic;              /* AccumPolicy::deterministic (ascending b) */
} evo_oracle_problem;

/* Returns 0 on success, 1 validation error, 2 numeric error (mirrors
 * ValidationError / NumericError of errors.hpp:15-30). */
int evo_oracle_forward(const evo_oracle_problem* p, const double* q, const double* k,
                       const double* v, const double* bias1, const double* bias2,
                       double* o, double* lse);

int evo_oracle_backward(const evo_oracle_problem* p, const double* q, const double* k,
                        const double* v, const double* bias1, const double* bias2,
                        const double* o, const double* lse, const double* dout,
                        double* dq, double* dk, double* dv, double* dbias1, double* dbias2);

/* Round a buffer onto the bf16 / f16 / f32 grid (RNE, saturating like
 * numeric_format.cpp:42-78); used to build identically-rounded inputs. */
void evo_oracle_round(double* x, int64_t n, int mantissa_bits, int exponent_bits);

/* Multi-threaded driver: rows of B are sharded over `threads` workers (the
 * reference is reentrant across problems); per-shard dbias2
 * partials are summed in ascending shard order. */
int evo_oracle_fwd_bwd_threaded(const evo_oracle_problem* p, int threads, const double* q,
                                const double* k, const double* v, const double* bias1,
                                const double* bias2, const double* dout, double* o,
                                double* lse, double* dq, double* dk, double* dv,
                                double* dbias2);

#ifdef __cplusplus
}
#endif
#endif
