# ncu --set full of one launch of a kernel (regex $1 on the DEMANGLED name, so template
# arguments can select an instance; skip $2) in one factorization step, warm caches,
# dense warp sampling. ncu prints template arguments as (int)64, (bool)0: use . for the parentheses:
# bash tools/ncu_kernel.sh 'k_gemm<.int.64, .int.64, .int.2, .int.4, .bool.0, .bool.1, .int.2, .int.1>' 2 out_name
python tools/profile_step.py --what factor > /dev/null 2>&1 || exit 1
ncu --set full --import-source on --warp-sampling-interval 0 --cache-control none --clock-control none \
  --profile-from-start off --kernel-name-base demangled -k regex:"$1" --launch-skip "$2" --launch-count 1 -o gpurun_out/"$3" \
  python tools/profile_step.py --what factor > gpurun_out/"$3".log 2>&1
tail -2 gpurun_out/"$3".log
