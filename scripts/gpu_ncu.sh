cd $GRAFT_REPO_ROOT
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$B > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-k1_correct|k3_filter|k_fft_mid}" -s ${NCU_S:-5} -c ${NCU_C:-3} -o gpurun_out/${NCU_O:-prof} $B > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full.log
