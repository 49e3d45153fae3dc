# usage: bash tools/_ab.sh <config> <what> ; compares lib/libevoattn_{old,new}.so on this box
for v in old new old new; do
  cp paper_2310_04610_b200/lib/libevoattn_$v.so paper_2310_04610_b200/lib/libevoattn.so
  timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab_$v.csv python tools/run_op.py --config $1 --what $2 --iters 3 > /dev/null 2>&1
  python -c "
import csv
rows=[r for r in csv.reader(open('gpurun_out/ab_$v.csv')) if len(r)>5]
hdr=rows[0]; ki=hdr.index('Kernel Name'); vi=hdr.index('Metric Value')
print('$v', [(r[ki].split('(')[0].split()[-1][:18], r[vi]) for r in rows if ('bk::' in r[ki] or 'evo::' in r[ki])][-8:])" >> gpurun_out/ab.txt
done
cp paper_2310_04610_b200/lib/libevoattn_new.so paper_2310_04610_b200/lib/libevoattn.so
