#!/bin/bash
# Libraries: ${LIBDIR:-abtest}/lib<V>.so, built with NVCC_EXTRA=... python paper_2304_03946_b200/build.py
# and copied there; FLEXMOE_B200_LIB makes the package load that build.
# A/B of two library builds on the same box: alternating bench runs.
for i in $(seq 1 ${ITERS:-3}); do
  for v in ${VARIANTS:-A B}; do
    FLEXMOE_B200_LIB=$PWD/${LIBDIR:-abtest}/lib$v.so timeout 300 python bench.py --steps 40 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; j=json.loads(sys.stdin.read()); k=j['kernels']; print('$v', round(j['value']/1e6,3), j['roofline']['frac'], j['clocks']['sm_mhz'], {n:round(k[n]['ms_per_step'],3) for n in k if n.startswith('ffn') or n in ('gate','dispatch','combine_fwd','combine_bwd','bias_grad','gate_wgrad','unpermute')})"
  done
done
