cd $GRAFT_REPO_ROOT
python scripts/probe_stages.py large > gpurun_out/probe.log 2>&1
python scripts/probe_stages.py realtime >> gpurun_out/probe.log 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
