# round 2 session 3, call X: final verification at the session tip (drain FADD2 + A-loop trims) — smoke, GPU suite, bench + reference arm, launch list, ncu of the BN=64 / BN=128 / stem levels
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? >> gpurun_out/status.txt
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$? >> gpurun_out/status.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-sweeps --cfg4-pop 0 --gen-pop 0 > gpurun_out/ncu_launch.log 2>&1; echo ncul=$? >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel --launch-skip 54 -c 1 -o gpurun_out/s3x_stem python scripts/conv_levels.py > gpurun_out/ncu_stem.log 2>&1; echo ncustem=$? >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel --launch-skip 59 -c 1 -o gpurun_out/s3x_l64 python scripts/conv_levels.py > gpurun_out/ncu_l64.log 2>&1; echo ncul64=$? >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel --launch-skip 99 -c 1 -o gpurun_out/s3x_l128 python scripts/conv_levels.py > gpurun_out/ncu_l128.log 2>&1; echo ncul128=$? >> gpurun_out/status.txt
