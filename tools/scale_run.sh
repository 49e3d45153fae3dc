# strong scaling of C4 (the config's rows split over the ranks) at 1, 2, 4 GPUs on one box
for n in 1 2 4; do
  if [ $n = 1 ]; then
    timeout 400 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/scale_n1.json 2> gpurun_out/scale_n1.err
  else
    timeout 400 python -m torch.distributed.run --nnodes 1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2960$n \
        bench.py --gpus $n --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/scale_n$n.json 2> gpurun_out/scale_n$n.err
  fi
  python -c "import json; d=json.loads(open('gpurun_out/scale_n$n.json').read().strip().splitlines()[-1]); print($n, round(d['value'],1), round(d['ms_per_step'],4), {k: round(v['ms'],4) for k,v in d['roofline']['kernels'].items()}, d['dbias2_allreduce_us'], d['e2e']['value'], (d.get('parity') or {}).get('pass'))"
done
timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 tools/mgpu_check.py > gpurun_out/mgpu4.log 2>&1
grep "PASS\|FAIL" gpurun_out/mgpu4.log
