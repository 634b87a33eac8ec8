# round 2, call M: per-tile A mode without row setup for TMA tiles; split corrections restored
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/levels.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_parity.log 2>&1; echo parity=$? >> gpurun_out/status.txt
for t in 1 0; do for args in "--prec fp32" "--prec bf16" "--fixture vgg16 --mode dimension --pop 8 --prec bf16"; do
  echo "== TMA=$t $args" >> gpurun_out/levels.txt
  TOBF_CONV_TMA=$t timeout 300 python scripts/conv_levels.py $args --order >> gpurun_out/levels.txt 2>&1
done; done
