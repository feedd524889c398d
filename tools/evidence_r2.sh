# Round-2 evidence on one B200. The plain bench runs first (no profiler); every
# ncu pass below is a separate run of tools/profile_step.py after that exited 0.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/r02_bench_cfg3.json 2> gpurun_out/r02_bench_cfg3.err || exit 1
python bench.py --impl reference > gpurun_out/r02_bench_reference_arm.json 2> gpurun_out/r02_bench_reference_arm.err
python bench.py --config cfg4 --no-cpu > gpurun_out/r02_bench_cfg4.json 2> gpurun_out/r02_bench_cfg4.err
python bench.py --config cfg5 --no-cpu > gpurun_out/r02_bench_cfg5.json 2> gpurun_out/r02_bench_cfg5.err
python tests/fullsize_parity.py --out gpurun_out/r02_fullsize_parity.json > gpurun_out/r02_fullsize_parity.log 2>&1
python tools/profile_step.py --what both > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r02_launches_step.csv python tools/profile_step.py --what both > gpurun_out/ncu_launch.log 2>&1
python tools/launch_summary.py gpurun_out/r02_launches_step.csv > gpurun_out/r02_launch_summary.txt
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r02_dram_factor.csv python tools/profile_step.py --what factor > gpurun_out/ncu_dram_f.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r02_dram_solve.csv python tools/profile_step.py --what solve > gpurun_out/ncu_dram_s.log 2>&1
python tools/dram_sum.py gpurun_out/r02_dram_factor.csv > gpurun_out/r02_dram_factor.txt
python tools/dram_sum.py gpurun_out/r02_dram_solve.csv > gpurun_out/r02_dram_solve.txt
# ncu --set full of the top kernels (names as ncu demangles them)
cap() {  # regex, skip, what, out
  ncu --set full --import-source on --clock-control none --profile-from-start off --kernel-name-base demangled \
    -k regex:"$1" --launch-skip "$2" --launch-count 1 -o gpurun_out/"$4" python tools/profile_step.py --what "$3" \
    > gpurun_out/"$4".log 2>&1
}
cap 'k_gemm<.int.128, .int.64, .int.4, .int.2, .bool.0, .bool.1, .int.3, .int.2>' 60 factor r02_ncu_leaf_update_trsm
cap 'k_gemm_group' 4 factor r02_ncu_group
cap 'k_potrf64' 40 factor r02_ncu_potrf
cap 'k_gemm<.int.64, .int.64, .int.2, .int.4, .bool.0, .bool.1, .int.2, .int.1>' 2 factor r02_ncu_gauss
cap 'k_leaf_bwd' 0 solve r02_ncu_leafbwd
cap 'k_node_up_cl' 0 solve r02_ncu_nodeup
ls -la gpurun_out | tail -40
