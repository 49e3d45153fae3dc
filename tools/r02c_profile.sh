# Final round-2 evidence for the shipped library at C4 (each capture after the same program exited 0
# without a profiler): bench launch list, ncu --set full of the forward and of the backward call
# (preamble, main kernel, conversion). Summaries into profiles/ are written on the box.
set -x
O=gpurun_out/r02c
mkdir -p $O
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 2 > $O/bench_pre.json 2>/dev/null && echo bench ok
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $O/launches_c4.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 1 > /dev/null 2>&1
python tools/ncu_summarize.py launches $O/launches_c4.csv $O/r02c_launches_c4.md --config c4 > /dev/null 2>&1
python tools/run_op.py --config c4 --iters 1 > /dev/null 2>&1 && echo run_op ok
cp profiles/ncu_traffic.json $O/ncu_traffic.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fwd_kernel" -c 1 \
    -o $O/full_fwd_c4 -f python tools/run_op.py --config c4 --iters 1 > $O/ncu_fwd.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bwd_kernel|prep_kernel|dq_convert" -c 3 \
    -o $O/full_bwd_c4 -f python tools/run_op.py --config c4 --what bwd --iters 1 > $O/ncu_bwd.log 2>&1
python tools/ncu_summarize.py full $O/full_fwd_c4.ncu-rep $O/r02c_ncu_full_fwd_c4.md --config c4 --traffic $O/ncu_traffic.json > /dev/null
python tools/ncu_summarize.py full $O/full_bwd_c4.ncu-rep $O/r02c_ncu_full_bwd_c4.md --config c4 --traffic $O/ncu_traffic.json > /dev/null
for r in fwd bwd; do
  ncu -i $O/full_${r}_c4.ncu-rep --page raw --csv > $O/raw_${r}_c4.csv 2>/dev/null
  ncu -i $O/full_${r}_c4.ncu-rep --page source --csv --print-source=sass > $O/src_${r}_c4.csv 2>/dev/null
done
du -sh $O
