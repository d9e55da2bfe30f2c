cd $GRAFT_REPO_ROOT
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
$B > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
$B > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k1_correct|k3_filter|k_fft_mid|k4_xifft" -s 5 -c 5 -o gpurun_out/prof_r1 $B > gpurun_out/ncu_full.log 2>&1
timeout 1200 python -m pytest tests -m "gpu and slow" -q > gpurun_out/pytest_slow.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_slow.log
