#!/bin/bash
# One ncu --set full capture (with source) of the kernels matching $KREGEX on
# the Large path (scripts/probe_stages.py run once plain first).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-k}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
P="python scripts/one_call.py ${CONFIG:-large} 3 - ${FLAGS:-0}"
$P > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"${KREGEX:-k3_}" -s ${SKIP:-1} -c ${COUNT:-1} -o gpurun_out/${TAG}_full $P > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${TAG}_ncu.log
