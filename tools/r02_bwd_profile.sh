# ncu --set full of the backward's main kernel (and preamble / conversion) at C4, C5, C2, C3
set -x
O=gpurun_out/r02b
mkdir -p $O
for cfg in c4 c5 c2 c3; do
  python tools/run_op.py --config $cfg --what bwd --iters 1 > /dev/null 2>&1 || echo "run_op $cfg failed"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bwd_kernel|prep_kernel|dq_convert" -c 3 \
      -o $O/full_bwd_$cfg -f python tools/run_op.py --config $cfg --what bwd --iters 1 > $O/ncu_$cfg.log 2>&1
  python tools/ncu_summarize.py full $O/full_bwd_$cfg.ncu-rep $O/r02_ncu_full_bwd_$cfg.md --config $cfg \
      --traffic $O/ncu_traffic.json > /dev/null 2>&1 || echo "summary $cfg failed"
  ncu -i $O/full_bwd_$cfg.ncu-rep --page raw --csv > $O/raw_bwd_$cfg.csv 2>/dev/null
  [ $cfg != c4 ] && rm -f $O/full_bwd_$cfg.ncu-rep
done
du -sh $O
