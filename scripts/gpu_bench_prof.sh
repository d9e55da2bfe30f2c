#!/bin/bash
# Round-2 measurement session: bench line (with e2e + CPU baseline), per-config
# stage times, the ncu launch list of the bench command, and one --set full
# capture of the five kernels (each after its command exited 0 without ncu).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-r2}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.log
for c in ${PROBE_CONFIGS:-tiny small freehand large realtime}; do timeout 300 python scripts/probe_stages.py $c >> gpurun_out/${TAG}_stages.txt 2>&1; done
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
if [ -z "$NO_NCU" ]; then
$B > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_|k_fft|k3_|k4_" --csv --log-file gpurun_out/${TAG}_launches.csv $B > gpurun_out/${TAG}_ncu_launch.log 2>&1
$B > gpurun_out/${TAG}_plain2.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k1_|k_fft|k3_|k4_" -s 15 -c 5 -o gpurun_out/${TAG}_full $B > gpurun_out/${TAG}_ncu_full.log 2>&1
fi
