#!/bin/bash
# Interleaved A/B of library builds on the configs[2..4] steps at N = 1 (torchrun, P2P phases):
# value, GEMM TFLOP/s, wgrad ms. VARIANTS="A B" WORKLOADS="cfg3 cfg5" ITERS=2 LIBDIR=abtest
for i in $(seq 1 ${ITERS:-2}); do
  for w in ${WORKLOADS:-cfg3 cfg4 cfg5}; do
    for v in ${VARIANTS:-A B}; do
      FLEXMOE_B200_LIB=$PWD/${LIBDIR:-abtest}/lib$v.so timeout 400 python -m torch.distributed.run --nnodes=1 \
        --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29617 bench.py --gpus 1 --workload $w \
        --steps ${STEPS:-30} --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; j=json.loads(sys.stdin.read()); k=j['kernels']
print('$w $v', round(j['value']/1e6,3), 'Mtok/s', j['clocks']['sm_mhz'], 'MHz gemm', j['roofline']['achieved'], 'wgrad ms', k.get('ffn2_wgrad',{}).get('ms_per_step'), k.get('ffn1_wgrad',{}).get('ms_per_step'),
      {n: round(k[n]['ms_per_step'], 4) for n in ('dispatch', 'combine_fwd', 'combine_bwd', 'unpermute', 'bias_grad') if n in k})"
    done
  done
done
