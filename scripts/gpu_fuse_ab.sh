#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu" -q -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
for c in large realtime freehand; do timeout 300 python scripts/probe_stages.py $c >> gpurun_out/probe.log 2>&1; SAR_NO_FUSE=1 timeout 300 python scripts/probe_stages.py $c 2>&1 | sed 's/^/nofuse /' >> gpurun_out/probe.log; done
