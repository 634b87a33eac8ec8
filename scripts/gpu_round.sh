# One GPU verification pass: smoke, GPU parity tests, bench, launch list, conv
# traffic capture and ncu full captures of the top kernels. Outputs in gpurun_out/.
set -x
rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? >> gpurun_out/status.txt
L=${CONV_LAUNCHES:-52}
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --print-units base -k regex:conv_tc_kernel --launch-skip $L -c $L --csv --log-file gpurun_out/conv_traffic.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-sweeps --cfg4-pop 0 > gpurun_out/ncu_traffic.log 2>&1; echo ncut=$? >> gpurun_out/status.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-sweeps --cfg4-pop 0 > gpurun_out/ncu_launch.log 2>&1; echo ncul=$? >> gpurun_out/status.txt
# full captures: a BN=64 stage-1 level (launch 4 of the step) and a BN=128 stage-4 level (launch 34)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel --launch-skip $((L + 4)) -c 1 -o gpurun_out/conv64_full python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-sweeps --cfg4-pop 0 > gpurun_out/ncu_full64.log 2>&1; echo ncuf64=$? >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel --launch-skip $((L + 34)) -c 1 -o gpurun_out/conv128_full python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-sweeps --cfg4-pop 0 > gpurun_out/ncu_full128.log 2>&1; echo ncuf128=$? >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:levenshtein_bp --launch-skip 12 -c 1 -o gpurun_out/ler_full python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --cfg4-pop 0 > gpurun_out/ncu_ler.log 2>&1; echo ncufl=$? >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lstm_ctc --launch-skip 3 -c 1 -o gpurun_out/lstm_full python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-sweeps --cfg4-pop 0 > gpurun_out/ncu_lstm.log 2>&1; echo ncuflstm=$? >> gpurun_out/status.txt
