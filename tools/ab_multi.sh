# usage: bash tools/ab_multi.sh <config> <what> v1 v2 ... ; times lib/libevoattn_<v>.so variants on this box (2 rounds)
out=gpurun_out/ab_multi.txt; : > $out
for round in 1 2; do
for v in "${@:3}"; do
  cp paper_2310_04610_b200/lib/libevoattn_$v.so paper_2310_04610_b200/lib/libevoattn.so
  timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/abm_$v.csv python tools/run_op.py --config $1 --what $2 --iters 3 > /dev/null 2>&1

done
done
python tools/ab_parse.py "${@:3}" | tee $out
