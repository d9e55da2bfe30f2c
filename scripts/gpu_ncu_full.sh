#!/bin/bash
# ncu --set full capture of the path's kernels on one bench step (after a clean run of the same command).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS}"
$B > gpurun_out/plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-k1_|k_fft|k3_|k4_}" -s ${NCU_S:-15} -c ${NCU_C:-5} -o gpurun_out/${NCU_O:-prof} -f $B > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full.log
