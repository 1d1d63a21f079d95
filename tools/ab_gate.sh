#!/bin/bash
# A/B of gate builds (resident CTAs per SM, NVCC_EXTRA=-DFM_GATE_CTAS=<n>):
# the gate phase alone (profiles/gate_microbench.py, L2 flushed) and in the
# configs[1] step (bench.py's live per-phase timing), interleaved.
for i in $(seq 1 ${ITERS:-2}); do
  for v in ${VARIANTS:-G2 G3 G4}; do
    for n in 16 64 128; do
      echo -n "$v "; FLEXMOE_B200_LIB=$PWD/${LIBDIR:-abtest}/lib$v.so timeout 120 python profiles/gate_microbench.py $n 2>&1 | tail -1
    done
    FLEXMOE_B200_LIB=$PWD/${LIBDIR:-abtest}/lib$v.so timeout 300 python bench.py --steps 40 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; j=json.loads(sys.stdin.read()); k=j['kernels']; print('$v step', round(j['value']/1e6,3), j['clocks']['sm_mhz'], k['gate'])"
  done
done
