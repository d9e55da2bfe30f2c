cd $GRAFT_REPO_ROOT
python scripts/probe_stages.py large > gpurun_out/probe.log 2>&1
python scripts/probe_stages.py realtime >> gpurun_out/probe.log 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${NCU_K}" -s ${NCU_S:-3} -c ${NCU_C:-2} -o gpurun_out/${NCU_O:-prof} $B > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full.log
