#!/bin/bash
# Round-end measurement session (each ncu capture only after its command ran
# cleanly without ncu): smoke, the bench line of the Large config with e2e and
# the oracle baseline, per-config stage times, the other modes' bench lines,
# the ncu launch list of the bench command, one --set full capture of the five
# kernels, and the whole GPU test suite.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${TAG:-r2f}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,power.limit --format=csv > gpurun_out/${T}_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench_large.log 2>&1; echo "bench rc=$?" >> gpurun_out/${T}_bench_large.log
for c in tiny small freehand large realtime; do timeout 300 python scripts/probe_stages.py $c >> gpurun_out/${T}_stage_times_all_configs.txt 2>&1; done
for a in "--config realtime" "--config freehand --grid nufft" "--config freehand --grid nearest" "--config large --stolt nufft" "--config large --planes 0.3,0.35"; do
  echo "== $a" >> gpurun_out/${T}_bench_modes.log
  timeout 600 python bench.py $a --steps 10 --warmup 3 --no-e2e --no-cpu-baseline >> gpurun_out/${T}_bench_modes.log 2>&1
done
if [ -z "$NO_NCU" ]; then
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$B > gpurun_out/${T}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_|k_fft|k3_|k4_" --csv --log-file gpurun_out/${T}_large_launches.csv $B > gpurun_out/${T}_ncu_launch.log 2>&1
echo "ncu launch rc=$?" >> gpurun_out/${T}_ncu_launch.log
P="python scripts/one_call.py large 2"
$P > gpurun_out/${T}_plain2.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k1_|k_fft|k3_|k4_" -s 5 -c 5 -o gpurun_out/${T}_full $P > gpurun_out/${T}_ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/${T}_ncu_full.log
fi
if [ -z "$NO_PYTEST" ]; then
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.txt
fi
