# ncu --set full of one launch of the fused leaf update+TRSM GEMM (factor step)
python tools/profile_step.py --what factor > /dev/null 2>&1 || exit 1
ncu --set full --import-source on --clock-control none --profile-from-start off \
  --kernel-name-base demangled -k regex:'k_gemm<.int.128, .int.64, .int.4, .int.2, .bool.0, .bool.1, .int.3, .int.2>' --launch-skip 14 --launch-count 1 \
  -o gpurun_out/ncu_top_gemm python tools/profile_step.py --what factor > gpurun_out/ncu_top.log 2>&1
tail -2 gpurun_out/ncu_top.log
