/* evoattn.h — C-ABI of the B200-native Evoformer attention (DS4Sci_EvoformerAttention).
 *
 * This is the drop-in boundary: plain pointers and sizes, no torch types.
 * Each entry point replaces one operator of the reference's API:
 *
 *   evo_attn_fwd   <- evomem::attn_forward_tiled
 *                     /root/reference/proj/core/include/evomem/attention_tiled.hpp:85-86
 *                     (implementation attention_tiled.cpp:57-180)
 *   evo_attn_bwd   <- evomem::attn_backward_tiled
 *                     attention_tiled.hpp:94-97 (attention_tiled.cpp:182-340)
 *   evo_attn_*_workspace_size  — device scratch the caller owns (the
 *                     reference's "tiled/work", "tiled/stats", "tiled/delta"
 *                     ledger allocations, attention_tiled.cpp:79-97, 229).
 *   evo_status     <- the reference's exception taxonomy errors.hpp:15-36
 *                     (ValidationError / NumericError / UsageError).
 *
 * Shapes follow DeepSpeed's DS4Sci_EvoformerAttention (north star):
 *   q, k, v, o, do, dq, dk, dv : [Bo, N, L, H, D]   (== reference (B, L, H, D), B = Bo*N)
 *   bias1 (mask)  / dbias1     : [Bo, N, 1, 1, L]   (optional; not in the reference)
 *   bias2 (pair)  / dbias2     : [Bo, 1, H, L, L]   (optional; reference `bias` (H, L, L) is Bo == 1)
 *   lse                         : [Bo*N, H, L] fp32, natural-log units
 *                                 (reference RowStats is (H, B, L); same values)
 * All pointers are DEVICE pointers owned by the caller; nothing is allocated
 * inside. Calls are stream-ordered and asynchronous. Contiguous row-major.
 */
#ifndef EVOATTN_H
#define EVOATTN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* evo_stream_t; /* == cudaStream_t */

typedef enum {
  EVO_OK = 0,
  EVO_ERR_VALIDATION = 1, /* ValidationError: shapes, dtypes, missing inputs, bad workspace */
  EVO_ERR_NUMERIC = 2,    /* NumericError: non-finite scale */
  EVO_ERR_USAGE = 3,      /* UsageError: API misuse (null descriptor, no device) */
  EVO_ERR_CUDA = 4,       /* a CUDA launch / runtime failure */
  EVO_ERR_UNSUPPORTED = 5 /* shape outside the kernels' envelope (e.g. D > 64 on fp32) */
} evo_status;

typedef enum { EVO_F32 = 0, EVO_BF16 = 1, EVO_F16 = 2 } evo_dtype;

/* Kernel family selection. AUTO picks tcgen05 (sm_100a tensor cores) for
 * bf16/f16 with D in {8, 16, 32, 64} (forward) and D in {8, 16, 32}, L % 8 == 0
 * (backward; D = 8 runs the D = 16 kernels on zero-padded TMA boxes), and the SIMT (FFMA) kernels otherwise
 * (fp32 must not use TF32: it fails the 1e-4 parity bar). */
typedef enum { EVO_PATH_AUTO = 0, EVO_PATH_SIMT = 1, EVO_PATH_TCGEN05 = 2 } evo_path;

typedef struct {
  int64_t Bo;        /* outer batch of the pair bias */
  int64_t N;         /* rows per outer batch (MSA rows / triangle start nodes) */
  int64_t L;         /* attended axis */
  int64_t H;         /* heads */
  int64_t D;         /* head dim */
  evo_dtype dtype;   /* dtype of q, k, v, o, do, dq, dk, dv, bias1, bias2 */
  double scale;      /* logit scale (reference default 1/sqrt(D), attention.cpp:43-45) */
  int has_bias1;     /* mask bias present */
  int has_bias2;     /* pair bias present */
  evo_dtype dbias_dtype; /* dtype of dbias1/dbias2 outputs: EVO_F32 = the reference's
                            UpcastF32 policy (attention_tiled.cpp:218-223), or == dtype */
  evo_path path;
  void* dbias2_multicast; /* backward, multi-GPU: NVSwitch multicast address of a symmetric fp32
                             dBias2 buffer (dbias2 = this rank's replica, dbias_dtype EVO_F32,
                             accumulate_dbias = 1). The kernel adds its partial through it, so every
                             rank's replica receives the sum of all ranks: the cross-GPU reduction
                             happens inside the kernel. The caller zeroes all replicas and
                             synchronises the ranks before and after the call. NULL = local only. */
  int need_dbias1;        /* backward: the call will ask for dbias1. Sizes the workspace for it (the
                             tcgen05 backward then splits the query axis into chunks of 2 tiles and
                             reduces dK/dV in fp32); a dbias1 request with need_dbias1 == 0 is a
                             ValidationError. The reference has no bias1: 0 there. */
  int axes_swapped;       /* 1 = q, k, v, o (and do, dq, dk, dv) are [L, N, H, D] — the raw
                             MSA-column / triangle-end-node layout whose attended axis is axis 0
                             (layout_from_msa, attention.cpp:109-119) — read and written in place
                             through the strides, no transposed copy. Requires Bo == 1; bias1, bias2,
                             lse and the dbias outputs stay canonical ([N, L], [H, L, L], [N, H, L]).
                             0 = canonical [Bo, N, L, H, D]. */
  int check_numerics;     /* 1 = NumericError contract of the reference (attention_tiled.cpp:49-65,
                             125-127, 209): the kernels flag NaN inputs (Q, K, V, biases, dO) and
                             non-finite logit rows (a NaN / non-finite LSE or delta, NaN outputs);
                             the call then synchronises its stream and returns EVO_ERR_NUMERIC.
                             Logits of -inf at some keys (masking) are allowed; a row with no finite
                             logit is flagged. 0 = no checks, fully asynchronous. */
  int deterministic;      /* backward: AccumPolicy::deterministic (attention_tiled.hpp:35-44; the
                             reference default): every cross-CTA reduction (dBias2, dBias1, dQ and
                             the chunked dK/dV) runs in a fixed order, so two runs are bit-identical
                             (SPEC.md:211). The SIMT backward is always ordered. 0 = unordered fp32
                             reductions (faster). */
  int has_gate;           /* OpenFold's sigmoid output gate fused into the operator (the _gated entry
                             points): o = sigmoid(G) * attention(q, k, v). Not in the reference
                             (SPEC.md:153 lists gating as a non-goal); SURVEY.md §8(f)3. */
} evo_attn_desc;

size_t evo_attn_fwd_workspace_size(const evo_attn_desc* desc);
size_t evo_attn_bwd_workspace_size(const evo_attn_desc* desc);

/* Forward: o = softmax(scale*q k^T + bias1 + bias2) v, lse = logsumexp per row.
 * bias1/bias2 may be NULL when the descriptor says absent. */
evo_status evo_attn_fwd(const evo_attn_desc* desc, const void* q, const void* k, const void* v,
                        const void* bias1, const void* bias2, void* o, float* lse,
                        void* workspace, size_t workspace_bytes, evo_stream_t stream);

/* Backward by recomputation from lse. dbias1/dbias2 may be NULL (not wanted).
 * dbias2 is the batch-axis sum of dS (reduced inside the kernels); when
 * accumulate_dbias != 0 it is ADDED to the caller's dbias2/dbias1 buffers
 * (dbias_dtype must be EVO_F32), which lets a row-sharded launcher
 * accumulate partial sums before its all-reduce. */
evo_status evo_attn_bwd(const evo_attn_desc* desc, const void* dout, const void* q, const void* k,
                        const void* v, const void* bias1, const void* bias2, const void* o,
                        const float* lse, void* dq, void* dk, void* dv, void* dbias1,
                        void* dbias2, int accumulate_dbias, void* workspace,
                        size_t workspace_bytes, evo_stream_t stream);

/* Fused output gate (desc.has_gate = 1; OpenFold gating). gate = G logits and
 * dgate in the layout of q / o. Forward: o = sigmoid(G) * softmax(...) v — the gate is applied in
 * the forward kernel's epilogue, so the ungated output is never stored. Backward: dout is the
 * gradient of the GATED output o (as the forward returned it); the preamble forms
 * dO = dout * sigmoid(G) for the attention backward and dgate = dout * o * (1 - sigmoid(G)) in the same
 * pass that computes delta = sum_d dout * o (the gate cancels in delta). */
evo_status evo_attn_fwd_gated(const evo_attn_desc* desc, const void* q, const void* k, const void* v,
                              const void* bias1, const void* bias2, const void* gate, void* o,
                              float* lse, void* workspace, size_t workspace_bytes, evo_stream_t stream);
evo_status evo_attn_bwd_gated(const evo_attn_desc* desc, const void* dout, const void* q, const void* k,
                              const void* v, const void* bias1, const void* bias2, const void* gate,
                              const void* o, const float* lse, void* dq, void* dk, void* dv, void* dgate,
                              void* dbias1, void* dbias2, int accumulate_dbias, void* workspace,
                              size_t workspace_bytes, evo_stream_t stream);

/* Which kernel family AUTO resolves to for this descriptor (EVO_PATH_SIMT or
 * EVO_PATH_TCGEN05); negative if the descriptor is invalid. */
int evo_attn_resolved_path(const evo_attn_desc* desc);

/* Which kernel family the BACKWARD resolves to (the tcgen05 backward's envelope is narrower than
 * the forward's: 16-bit, D in {16, 32}, L % 8 == 0); negative if invalid or an explicit
 * EVO_PATH_TCGEN05 request cannot be honoured. */
int evo_attn_resolved_bwd_path(const evo_attn_desc* desc);

/* Number of kernel launches the last fwd / bwd call issued on this thread. */
int evo_attn_last_launch_count(void);

/* Message of the last error on this thread ("" if none). */
const char* evo_attn_last_error(void);

/* Host-side synthetic inputs identical to the reference's instance generator (not the hot path):
 * draws [skip, skip + n) of the stream derived_rng(seed, stream) — SeededRng (std::mt19937_64, top 53
 * bits; rng.hpp:16-43) — as lo + (hi - lo) * uniform(), rounded RNE to `dtype` exactly like
 * random_uniform / round_to_format (rng.cpp:5-10, numeric_format.cpp:42-78), into HOST memory.
 * random_problem (run.cpp:178-189) draws Q, K, V, then the bias from one stream; the harness's dO
 * comes from stream + 2^20 (run.cpp:194-195). */
evo_status evo_random_uniform(uint64_t seed, uint64_t stream, int64_t skip, int64_t n, double lo,
                              double hi, evo_dtype dtype, void* host_out);

/* DS4Sci mask bias1 (no reference counterpart): for rows [row0, row0 + rows) of an [*, L] mask, one
 * uniform draw per (row, key) of derived_rng(seed, stream); value `neg` where draw < rate, else 0;
 * key 0 is never masked (no fully masked row). HOST memory, `dtype` elements. */
evo_status evo_random_mask(uint64_t seed, uint64_t stream, int64_t rows, int64_t row0, int64_t L,
                           double rate, double neg, evo_dtype dtype, void* host_out);

/* Pair-bias projection feeding bias2 (no reference counterpart — OpenFold's
 * MSARowAttentionWithPairBias layer_norm_z + linear_z, SPEC.md:153 lists it as a non-goal):
 *   bias2[b, 0, h, i, j] = sum_c LN(z[b, i, j, :])_c * w[c, h],  LN(x) = (x - mean) / sqrt(var + eps) * ln_w + ln_b
 * z [Bo, L, L, C] (bf16 / f16), ln_w / ln_b [C] fp32, w [C, H] fp32 (nn.Linear(C, H).weight transposed);
 * bias2 [Bo, 1, H, L, L] in z's dtype — the layout evo_attn_fwd / evo_attn_bwd read. The backward takes
 * dbias2 in that same layout (fp32 — evo_attn_bwd's UpcastF32 output — or z's dtype) and writes dz (z's
 * dtype) and fp32 dln_w, dln_b, dw (per-CTA partials in the caller's workspace, summed in a fixed order:
 * deterministic). Envelope: C a multiple of 32 up to 256, H <= 16. */
typedef struct {
  int64_t Bo, L, C, H;
  evo_dtype dtype;       /* z, bias2, dz */
  evo_dtype dbias_dtype; /* the backward's dbias2 input: EVO_F32 or dtype */
  float eps;
} evo_pair_bias_desc;

evo_status evo_pair_bias_fwd(const evo_pair_bias_desc* desc, const void* z, const float* ln_w, const float* ln_b,
                             const float* w, void* bias2, evo_stream_t stream);
size_t evo_pair_bias_bwd_workspace_size(const evo_pair_bias_desc* desc);
evo_status evo_pair_bias_bwd(const evo_pair_bias_desc* desc, const void* dbias2, const void* z, const float* ln_w,
                             const float* ln_b, const float* w, void* dz, float* dln_w, float* dln_b, float* dw,
                             void* workspace, size_t workspace_bytes, evo_stream_t stream);

/* Library version string, e.g. "evoattn 0.1 sm_100a". */
const char* evo_attn_version(void);

#ifdef __cplusplus
}
#endif
#endif /* EVOATTN_H */
