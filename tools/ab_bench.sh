# usage: bash tools/ab_bench.sh v1 v2 ... ; bench.py C4 with lib/libevoattn_<v>.so swapped in, twice each
for rep in 1 2; do for v in "$@"; do
  cp paper_2310_04610_b200/lib/libevoattn_$v.so paper_2310_04610_b200/lib/libevoattn.so
  touch paper_2310_04610_b200/lib/libevoattn.so
  echo -n "$v "; timeout 300 python bench.py --no-cpu-baseline --e2e-steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],4), {k: round(v['ms'],4) for k,v in d['roofline']['kernels'].items()})"
done; done
