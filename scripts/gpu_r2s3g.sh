# round 2 session 3, call G: ncu full (with source) of a BN=64 3x3 level (launch 5) at the tip
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel --launch-skip 59 -c 1 -o gpurun_out/s3_l64 python scripts/conv_levels.py > gpurun_out/ncu_l64.log 2>&1; echo ncul64=$? >> gpurun_out/status.txt
