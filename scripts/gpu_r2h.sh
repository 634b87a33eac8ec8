# round 2, call H: ncu full of conv launch 1 (1x1 on 112^2) and 0 (stem); e2e micro-batch sweep at P=32
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel --launch-skip 53 -c 1 -o gpurun_out/conv_l1 python scripts/conv_levels.py > gpurun_out/ncu_l1.log 2>&1; echo ncu1=$? >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel --launch-skip 52 -c 1 -o gpurun_out/conv_l0 python scripts/conv_levels.py > gpurun_out/ncu_l0.log 2>&1; echo ncu0=$? >> gpurun_out/status.txt
for m in auto 8 8,8,16 4,12,16; do echo "== $m" >> gpurun_out/timeline_sweep.txt; timeout 300 python scripts/e2e_timeline.py 32 $m 2>&1 | grep -E "total|device|apply_plan" >> gpurun_out/timeline_sweep.txt; done
