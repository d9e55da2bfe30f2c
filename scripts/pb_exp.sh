#!/bin/bash
# fused pass-B experiments: times + ncu DRAM bytes for TMA vs plain S/I loads, with/without discard
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in "" "SAR_PB_PLAIN=1" "SAR_PB_PLAIN=1 SAR_NO_DISCARD=1"; do
  echo "== $v" >> gpurun_out/pb.log
  env SAR_FUSE=1 $v timeout 300 python scripts/probe_stages.py large 2>&1 | grep " comp" >> gpurun_out/pb.log
  env SAR_FUSE=1 $v timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_passb -c 1 python scripts/probe_stages.py large 2>&1 | grep -E "dram__|gpu__time" >> gpurun_out/pb.log
done
