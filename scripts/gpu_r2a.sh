# round 2, call A: full-size parity tests, cfg5 LSTM timing + ncu full capture of the real cfg5 launch
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
nproc > gpurun_out/nproc.txt; free -g >> gpurun_out/nproc.txt
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q --durations=0 > gpurun_out/pytest_full.log 2>&1; echo full=$? >> gpurun_out/status.txt
timeout 300 python scripts/cfg5_lstm.py > gpurun_out/cfg5.log 2>&1; echo cfg5=$? >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lstm_ctc --launch-skip 1 -c 1 -o gpurun_out/lstm512_full python scripts/cfg5_lstm.py --hidden 512 --reps 1 > gpurun_out/ncu_lstm512.log 2>&1; echo ncu512=$? >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lstm_ctc --launch-skip 1 -c 1 -o gpurun_out/lstm128_full python scripts/cfg5_lstm.py --hidden 128 --reps 1 > gpurun_out/ncu_lstm128.log 2>&1; echo ncu128=$? >> gpurun_out/status.txt
