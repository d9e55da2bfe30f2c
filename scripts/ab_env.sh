#!/bin/bash
# A/B of an environment switch on the per-stage times: AB_VAR=NAME AB_VALS="v1 v2" AB_CONFIGS="large freehand"
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
: > gpurun_out/ab.log
for rep in 1 2; do
for val in ${AB_VALS:-""}; do
  for c in ${AB_CONFIGS:-large}; do
    if [ "$val" = "-" ]; then unset $AB_VAR; else export $AB_VAR=$val; fi
    echo "== $AB_VAR=$val $c" >> gpurun_out/ab.log
    timeout 300 python scripts/probe_stages.py $c 2>&1 | head -1 >> gpurun_out/ab.log
  done
done
done
