# round 2 session 2: LSTM 8 traces per thread (r8w4 / r8w8) vs 4 (rb4 / rb8): bit-exact + cfg5 timing
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/lstm_variants.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -k "lstm or cfg5" > gpurun_out/pytest_lstm.log 2>&1; echo lstm=$? >> gpurun_out/status.txt
for rep in 1 2; do
for v in default rb4 rb8 r8w4 r8w8; do
  echo "== $v rep$rep" >> gpurun_out/lstm_variants.txt
  TOBF_LSTM_VARIANT=$v timeout 300 python scripts/cfg5_lstm.py >> gpurun_out/lstm_variants.txt 2>&1
done
done
for v in 1 0; do
  TOBF_INPUT_IM2COL=$v timeout 600 python bench.py --no-sweeps --cfg4-pop 0 --gen-pop 0 --no-cpu-baseline > gpurun_out/bench_x$v.json 2> gpurun_out/bench_x$v.err; echo bench_x$v=$? >> gpurun_out/status.txt
done
