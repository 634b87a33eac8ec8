# round 2, call E: LSTM register-blocked kernel (parity + cfg5 timing vs the round-1 kernel), full GPU suite
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "lstm or population or smoke" > gpurun_out/pytest_lstm.log 2>&1; echo lstm=$? >> gpurun_out/status.txt
timeout 300 python scripts/cfg5_lstm.py > gpurun_out/cfg5_rb.log 2>&1; echo cfg5=$? >> gpurun_out/status.txt
TOBF_LSTM_VARIANT=cluster16 timeout 300 python scripts/cfg5_lstm.py > gpurun_out/cfg5_old.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo gpu=$? >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lstm_ctc_rb --launch-skip 1 -c 1 -o gpurun_out/lstm512_rb python scripts/cfg5_lstm.py --hidden 512 --reps 1 > gpurun_out/ncu_lstm512.log 2>&1; echo ncu=$? >> gpurun_out/status.txt
