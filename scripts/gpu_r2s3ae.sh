# round 2 session 3, call AE: ncu full captures of the final tip's stem and BN=64 levels, and the launch list of a bench step
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel --launch-skip 54 -c 1 -o gpurun_out/s3f_stem python scripts/conv_levels.py > gpurun_out/ncu_stem.log 2>&1; echo ncustem=$? >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel --launch-skip 59 -c 1 -o gpurun_out/s3f_l64 python scripts/conv_levels.py > gpurun_out/ncu_l64.log 2>&1; echo ncul64=$? >> gpurun_out/status.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-sweeps --cfg4-pop 0 --gen-pop 0 > gpurun_out/ncu_launch.log 2>&1; echo ncul=$? >> gpurun_out/status.txt
