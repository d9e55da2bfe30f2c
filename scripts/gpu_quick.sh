#!/bin/bash
# parity suite + a quick bench line (no e2e / cpu baseline) + per-stage probe
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu" -q -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
for c in ${PROBE_CONFIGS:-realtime freehand}; do timeout 300 python scripts/probe_stages.py $c >> gpurun_out/probe.log 2>&1; done
