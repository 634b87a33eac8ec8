# round 2 session 2: bench at the tip (input-im2col stem), launch list, ncu of the new stem level + a BN=64 level
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? >> gpurun_out/status.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-sweeps --cfg4-pop 0 --gen-pop 0 > gpurun_out/ncu_launch.log 2>&1; echo ncul=$? >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel --launch-skip 52 -c 1 -o gpurun_out/conv_stem_im2col python scripts/conv_levels.py > gpurun_out/ncu_stem.log 2>&1; echo ncustem=$? >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel --launch-skip 56 -c 1 -o gpurun_out/conv_l4 python scripts/conv_levels.py > gpurun_out/ncu_l4.log 2>&1; echo ncul4=$? >> gpurun_out/status.txt
