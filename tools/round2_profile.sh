# Round-2 evidence run on one B200 (each command after the same program exited 0 without a profiler):
# launch list of the C4 bench, ncu --set full of the forward / backward kernels at C4, C5, C2, C3 and
# a D = 8 shape, compute-sanitizer memcheck / synccheck on three small shapes.
set -x
O=gpurun_out/r02
mkdir -p $O
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 2 > $O/bench_pre.json 2>/dev/null && echo bench ok
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file $O/launches_c4.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-parity --e2e-steps 1 > /dev/null 2>&1
for cfg in c4 c5 c2 c3; do
  python tools/run_op.py --config $cfg --iters 1 > /dev/null 2>&1 || echo "run_op $cfg failed"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fwd_kernel|bwd_kernel" -c 2 \
      -o $O/full_$cfg -f python tools/run_op.py --config $cfg --iters 1 > $O/ncu_$cfg.log 2>&1
done
timeout 600 ncu --set full --clock-control none -k regex:"fwd_kernel|dkdv_kernel|dq_kernel|delta_kernel" -c 4 \
    -o $O/full_d8 -f python tools/run_op.py --shape 1,512,384,8,8 --iters 1 > $O/ncu_d8.log 2>&1
for shp in 1,4,130,2,32 1,4,256,2,32 1,2,640,2,32; do
  for tool in memcheck synccheck; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/run_op.py --shape $shp --iters 1 \
        > $O/sanitizer_${tool}_${shp//,/x}.log 2>&1
    echo "$tool $shp rc=$?" >> $O/sanitizer_summary.txt
  done
done
ls -la $O
# summaries on the box (the reports are large): key counters per kernel, traffic merged for bench.py
for cfg in c4 c5 c2 c3 d8; do
  python tools/ncu_summarize.py full $O/full_$cfg.ncu-rep $O/r02_ncu_full_$cfg.md --config $cfg \
      --traffic $O/ncu_traffic.json > /dev/null 2>&1 || echo "summary $cfg failed"
  ncu -i $O/full_$cfg.ncu-rep --page raw --csv > $O/raw_$cfg.csv 2>/dev/null
  [ $cfg != c4 ] && rm -f $O/full_$cfg.ncu-rep
done
python tools/ncu_summarize.py launches $O/launches_c4.csv $O/r02_launches_c4.md --config c4 > /dev/null 2>&1
head -c 600 $O/sanitizer_memcheck_1x4x256x2x32.log
du -sh $O
