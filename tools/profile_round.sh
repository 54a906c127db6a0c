#!/bin/bash
# Round profile of the bench's default workload (cfg4 training minibatch), run on a GPU box:
#   1. plain run (must exit 0 first)
#   2. launch list of ONE eager step (the bench's profile_step NVTX range)
#   3. ncu --set full of the top kernels inside that step (dram traffic, stalls),
#      including the TMA-staged key-switch inner product
#   4. DRAM bytes per launch of every kernel of the step
set -e
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 > gpurun_out/prof_plain.log 2>&1
BENCH_NVTX=1 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx \
    --nvtx-include "profile_step/" --csv --log-file gpurun_out/launches_train.csv \
    python bench.py --steps 1 --warmup 3 > gpurun_out/prof_launches.log 2>&1
BENCH_NVTX=1 ncu --set full --clock-control none --import-source on --nvtx \
    --nvtx-include "profile_step/" --kernel-name-base demangled \
    -k regex:"k_ntt_cols_r<\(int\)8, \(bool\)0, \(int\)2|k_ntt_blocks_r<\(int\)8, \(bool\)0|k_bsgs_mma|k_ks_ip_rot<\(int\)1|k_ks_ip_rot_tma" -c 10 \
    -o gpurun_out/prof_train python bench.py --steps 1 --warmup 3 > gpurun_out/prof_full.log 2>&1
BENCH_NVTX=1 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx \
    --nvtx-include "profile_step/" --csv --log-file gpurun_out/dram_train.csv \
    python bench.py --steps 1 --warmup 3 > gpurun_out/prof_dram.log 2>&1
