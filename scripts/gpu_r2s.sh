# round 2, call S: epilogue L2 prefetch (conv), relaxed barrier A (LSTM), e2e micro splits
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/levels.txt gpurun_out/e2e_split.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_parity.log 2>&1; echo parity=$? >> gpurun_out/status.txt
for args in "--prec fp32" "--prec bf16" "--fixture vgg16 --mode dimension --pop 8 --prec bf16"; do
  echo "== $args" >> gpurun_out/levels.txt
  timeout 300 python scripts/conv_levels.py $args --order 2>&1 | head -8 >> gpurun_out/levels.txt
done
timeout 300 python scripts/cfg5_lstm.py > gpurun_out/cfg5.txt 2>&1; echo cfg5=$? >> gpurun_out/status.txt
for m in auto 16 12,12,8 12,20 10,12,10 16,8,8; do echo "== $m" >> gpurun_out/e2e_split.txt; timeout 300 python scripts/e2e_timeline.py 32 $m 2>&1 | grep -E "total" >> gpurun_out/e2e_split.txt; done
