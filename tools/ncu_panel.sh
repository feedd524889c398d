# ncu of one lu_panel launch at a top level (launch 300 of the factorization) and one at level 0
set -x
python tools/profile_step.py --what factor > gpurun_out/ps.log 2>&1 || exit 1
ncu --set full --import-source on --warp-sampling-interval 0 --clock-control none --profile-from-start off -k regex:k_lu_panel --launch-skip 300 --launch-count 1 -o gpurun_out/ncu_panel_top python tools/profile_step.py --what factor > gpurun_out/ncu1.log 2>&1
if [ "$1" = "both" ]; then
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_lu_panel --launch-skip 5 --launch-count 1 -o gpurun_out/ncu_panel_l0 python tools/profile_step.py --what factor > gpurun_out/ncu2.log 2>&1
fi
