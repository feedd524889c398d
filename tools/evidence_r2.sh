# Round-2 evidence on one B200 (run after the plain bench exited 0): the launch
# list of one factor+solve step, DRAM bytes of one factorization and one q=1
# solve, and ncu --set full captures of the top kernels.
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r02_launches_step.csv python tools/profile_step.py --what both > gpurun_out/ncu_launch.log 2>&1
python tools/launch_summary.py gpurun_out/r02_launches_step.csv > gpurun_out/r02_launch_summary.txt
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r02_dram_factor.csv python tools/profile_step.py --what factor > gpurun_out/ncu_dram_f.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/r02_dram_solve.csv python tools/profile_step.py --what solve > gpurun_out/ncu_dram_s.log 2>&1
python tools/dram_sum.py gpurun_out/r02_dram_factor.csv > gpurun_out/r02_dram_factor.txt
python tools/dram_sum.py gpurun_out/r02_dram_solve.csv > gpurun_out/r02_dram_solve.txt
ncu --set full --import-source on --clock-control none --profile-from-start off \
  -k regex:'k_gemm<128, 64, 4, 2, false, true, 3, 2>' --launch-skip 7 --launch-count 1 \
  -o gpurun_out/r02_ncu_leaf_gemm python tools/profile_step.py --what factor > gpurun_out/ncu_top.log 2>&1
ncu --set full --import-source on --clock-control none --profile-from-start off \
  -k regex:k_gemm_group --launch-skip 4 --launch-count 1 \
  -o gpurun_out/r02_ncu_group python tools/profile_step.py --what factor > gpurun_out/ncu_grp.log 2>&1
ncu --set full --import-source on --clock-control none --profile-from-start off \
  -k regex:k_leaf_bwd --launch-count 1 -o gpurun_out/r02_ncu_leafbwd python tools/profile_step.py --what solve > gpurun_out/ncu_bwd.log 2>&1
ncu --set full --import-source on --clock-control none --profile-from-start off \
  -k regex:k_node_up_cl --launch-count 1 -o gpurun_out/r02_ncu_nodeup python tools/profile_step.py --what solve > gpurun_out/ncu_nodeup.log 2>&1
ls -la gpurun_out | tail -20
