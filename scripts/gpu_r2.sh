#!/bin/bash
# round-2 GPU session: quick bench line, per-stage probes, then the parity suite
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
for c in ${PROBE_CONFIGS:-large realtime freehand}; do timeout 300 python scripts/probe_stages.py $c >> gpurun_out/probe.log 2>&1; done
if [ -z "$NO_PYTEST" ]; then
timeout ${PYTEST_TIMEOUT:-1500} python -m pytest tests -m "gpu" -q ${PYTEST_K:+-k "$PYTEST_K"} ${PYTEST_EXTRA} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
