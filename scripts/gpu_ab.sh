#!/bin/bash
# A/B per-kernel times of library variants: AB_CONFIGS x AB_LIBS (NAME:PATH ...)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-ab}
for rep in 1 2; do
for c in ${AB_CONFIGS:-large}; do
  timeout 600 python scripts/ab_variants.py $c ${AB_LIBS} >> gpurun_out/${TAG}.txt 2>&1
done
done
