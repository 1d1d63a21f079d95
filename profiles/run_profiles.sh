#!/bin/bash
# Recipe for the committed ncu evidence (run on the B200 via gpurun; 1 GPU):
#   launches list of one bench step (11 launches at configs[1]; cold-cache, serialised: compare
#   SHARES; summarize.py keeps the launches from one gate launch to the next)
#   --set full captures of the six grouped-GEMM launches and the HBM kernels
# Output in gpurun_out/; profiles/summarize.py turns it into profiles/*.md|json.
set -e
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -s 30 -c 40 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:grouped_gemm -s 18 -c 6 \
    -o gpurun_out/prof_gemm -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_gemm.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"gate_kernel|dispatch_kernel|dispatch_pipe|combine_fwd|combine_bwd|unpermute|segment_tile|expert_scan|plan_kernel" \
    -s 15 -c 5 -o gpurun_out/prof_hbm -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_hbm.log 2>&1
ncu --target-processes all --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/dist_launches.csv python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 \
    --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus 1 --workload cfg3 --steps 3 --warmup 3 \
    --no-cpu-baseline > gpurun_out/ncu_dist.log 2>&1
