# round 2, call V: LSTM gate loop with FFMA2 (fp32 pairs) — bit-exact parity + cfg5 timing + ncu
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "lstm or population or smoke or cfg5" > gpurun_out/pytest_lstm.log 2>&1; echo lstm=$? >> gpurun_out/status.txt
timeout 300 python scripts/cfg5_lstm.py > gpurun_out/cfg5_ffma2.log 2>&1; echo cfg5=$? >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lstm_ctc_rb --launch-skip 1 -c 1 -o gpurun_out/lstm512_ffma2 python scripts/cfg5_lstm.py --hidden 512 --reps 1 > gpurun_out/ncu_lstm512.log 2>&1; echo ncu=$? >> gpurun_out/status.txt
