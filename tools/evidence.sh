# Round evidence on one B200: bench line, per-launch list of one factor+solve
# step (ncu, cold-cache serialized), ncu --set full of the top factor kernel.
set -x
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_step.csv python tools/profile_step.py --what both > gpurun_out/ncu_launch.log 2>&1
python tools/launch_summary.py gpurun_out/launches_step.csv > gpurun_out/launch_summary.txt
ncu --set full --import-source on --clock-control none --profile-from-start off \
  --kernel-name-base demangled -k regex:'k_gemm<.int.128, .int.64, .int.4, .int.2, .bool.0, .bool.1, .int.3, .int.2>' --launch-skip 7 --launch-count 1 \
  -o gpurun_out/ncu_top_gemm python tools/profile_step.py --what factor > gpurun_out/ncu_top.log 2>&1
ncu --set full --import-source on --clock-control none --profile-from-start off \
  -k regex:k_leaf_bwd --launch-count 1 -o gpurun_out/ncu_leafbwd python tools/profile_step.py --what solve > gpurun_out/ncu_bwd.log 2>&1
ncu --set full --import-source on --clock-control none --profile-from-start off \
  -k regex:k_lu_slab --launch-skip 2 --launch-count 1 -o gpurun_out/ncu_slab python tools/profile_step.py --what factor > gpurun_out/ncu_slab.log 2>&1
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ls -la gpurun_out
