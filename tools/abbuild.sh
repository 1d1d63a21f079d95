#!/bin/bash
# Build library variants for an A/B: tools/abbuild.sh NAME "NVCC flags" [NAME "flags"]...
# Each lands in ${LIBDIR:-abtest}/lib<NAME>.so (the default build is restored after).
set -e
mkdir -p ${LIBDIR:-abtest}
while [ $# -ge 2 ]; do
  NVCC_EXTRA="$2" python paper_2304_03946_b200/build.py >/dev/null
  cp paper_2304_03946_b200/libflexmoe_b200.so ${LIBDIR:-abtest}/lib$1.so
  touch paper_2304_03946_b200/csrc/*.cu paper_2304_03946_b200/csrc/*.cpp  # force the next variant to recompile
  shift 2
done
python paper_2304_03946_b200/build.py >/dev/null
