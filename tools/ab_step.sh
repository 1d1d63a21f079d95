#!/bin/bash
# Interleaved A/B of library builds on the configs[1] step (bench.py live
# per-phase timing): value, gate, unpermute, tile sums, wgrads, clocks.
for i in $(seq 1 ${ITERS:-3}); do
  for v in ${VARIANTS:-A B}; do
    FLEXMOE_B200_LIB=$PWD/${LIBDIR:-abtest}/lib$v.so timeout 300 python bench.py --steps ${STEPS:-40} --no-cpu-baseline ${BENCH_ARGS} 2>/dev/null | tail -1 | python -c "
import json,sys; j=json.loads(sys.stdin.read()); k=j['kernels']
print('$v', round(j['value']/1e6,3), 'Mtok/s', j['clocks']['sm_mhz'], 'MHz', {n: (k[n]['ms_per_step']*1e3 if 'frac_hbm' not in k[n] else (round(k[n]['ms_per_step']*1e3,1), k[n]['frac_hbm'])) for n in k if n in ('gate','scan','route','unpermute','bias_grad','ffn2_wgrad','ffn1_wgrad','combine_bwd','dispatch')})"
  done
done
