for n in 2 4; do
  for mode in default c4 c8; do
    case $mode in default) ENVS="";; c4) ENVS="NCCL_MAX_CTAS=4";; c8) ENVS="NCCL_MAX_CTAS=8";; esac
    env $ENVS timeout 300 python -m torch.distributed.run --nnodes 1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2970$n \
      bench.py --gpus $n --steps 50 --warmup 5 --no-cpu-baseline --no-parity --e2e-steps 2 > gpurun_out/nccl_${mode}_$n.json 2> gpurun_out/nccl_${mode}_$n.err
    python -c "import json; d=json.loads(open('gpurun_out/nccl_${mode}_$n.json').read().strip().splitlines()[-1]); print($n, '$mode', round(d['value'],1), round(d['ms_per_step'],4), d['dbias2_allreduce_us'])" 2>&1 | tail -1
  done
done
