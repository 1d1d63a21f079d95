#!/bin/bash
# Libraries: ${LIBDIR:-abtest}/lib<V>.so, built with NVCC_EXTRA=... python paper_2304_03946_b200/build.py
# and copied there; FLEXMOE_B200_LIB makes the package load that build.
# A/B of library builds on the DistArm (configs[2] shapes) at the given Zipf exponents.
port=29700
for i in 1 2; do
  for z in ${ZIPFS:-0.0 1.25}; do
    for v in ${VARIANTS:-A B}; do
      port=$((port+1))
      ZIPF=$z FLEXMOE_B200_LIB=$PWD/${LIBDIR:-abtest}/lib$v.so timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port $port tools/zipf_probe.py --gpus 1 --workload cfg3 --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; j=json.loads(sys.stdin.read()); k=j['kernels']; print('$v', $z, round(j['value']/1e6,3), j['clocks']['sm_mhz'], {n:round(k[n]['ms_per_step'],3) for n in k if n.startswith('ffn') or n in ('bias_grad','combine_bwd','dispatch')})"
    done
  done
done
