#!/bin/bash
# Build library variants for an A/B: tools/abbuild.sh NAME "NVCC flags" [NAME "flags"]...
# Each lands in ${LIBDIR:-abtest}/lib<NAME>.so (the default build is restored after).
# Every variant recompiles every source (the incremental build only looks at timestamps).
set -e
mkdir -p ${LIBDIR:-abtest}
while [ $# -ge 2 ]; do
  touch paper_2304_03946_b200/csrc/*.cu paper_2304_03946_b200/csrc/*.cpp
  NVCC_EXTRA="$2" python paper_2304_03946_b200/build.py >/dev/null
  cp paper_2304_03946_b200/libflexmoe_b200.so ${LIBDIR:-abtest}/lib$1.so
  shift 2
done
touch paper_2304_03946_b200/csrc/*.cu paper_2304_03946_b200/csrc/*.cpp
python paper_2304_03946_b200/build.py >/dev/null
