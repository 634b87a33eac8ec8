# round 2, call L: per-tile A mode (TMA for Cp%32==0, cp.async otherwise, one launch per level)
# + merged tf32 correction accumulators (no per-tile correction slot)
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/levels.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "conv or execute or equivalence or derived or bf16 or population" > gpurun_out/pytest_parity.log 2>&1; echo parity=$? >> gpurun_out/status.txt
for args in "--prec fp32" "--prec bf16" "--fixture vgg16 --mode dimension --pop 8 --prec bf16"; do
  echo "== $args" >> gpurun_out/levels.txt
  timeout 300 python scripts/conv_levels.py $args --order >> gpurun_out/levels.txt 2>&1
done
echo "== split-corr build fp32" >> gpurun_out/levels.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --gen-pop 0 --cfg4-pop 0 --no-sweeps > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo bench=$? >> gpurun_out/status.txt
TOBF_CONV_TMA=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --gen-pop 0 --cfg4-pop 0 --no-sweeps --no-e2e > gpurun_out/bench_quick_cpasync.json 2>> gpurun_out/bench_quick.err
