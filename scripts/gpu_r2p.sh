# round 2, call P: mixed-mode lockstep fix; VGG bf16 + cfg4; parity; RN18 levels
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/levels.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_parity.log 2>&1; echo parity=$? >> gpurun_out/status.txt
for args in "--fixture vgg16 --mode dimension --pop 8 --prec bf16" "--fixture vgg16 --mode dimension --pop 8 --prec fp32" "--prec fp32" "--prec bf16"; do
  echo "== $args" >> gpurun_out/levels.txt
  timeout 300 python scripts/conv_levels.py $args --order 2>&1 | head -3 >> gpurun_out/levels.txt
done
timeout 900 python -c "
import json, sys
sys.argv=['bench.py']
import bench
a = bench.parse()
peaks = json.load(open('MEASURED_PEAKS.json')) if __import__('os').path.exists('MEASURED_PEAKS.json') else {}
print(json.dumps(bench.workload_cfg4(a, peaks)))
" > gpurun_out/cfg4.json 2> gpurun_out/cfg4.err; echo cfg4=$? >> gpurun_out/status.txt
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -x > gpurun_out/pytest_full.log 2>&1; echo full=$? >> gpurun_out/status.txt
