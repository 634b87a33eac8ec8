# One GPU verification pass: smoke, GPU parity tests, bench, launch list, conv
# traffic capture and ncu full captures of the top kernels. Outputs in gpurun_out/.
set -x
rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? >> gpurun_out/status.txt
L=${CONV_LAUNCHES:-52}
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --print-units base -k regex:conv_tf32x3 --launch-skip $L -c $L --csv --log-file gpurun_out/conv_traffic.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-sweeps > gpurun_out/ncu_traffic.log 2>&1; echo ncut=$? >> gpurun_out/status.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-sweeps > gpurun_out/ncu_launch.log 2>&1; echo ncul=$? >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:levenshtein_bp --launch-skip 12 -c 1 -o gpurun_out/ler_full python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --ler-pairs 10000000 > gpurun_out/ncu_ler.log 2>&1; echo ncufl=$? >> gpurun_out/status.txt
