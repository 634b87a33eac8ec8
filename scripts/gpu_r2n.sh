# round 2, call N: vectorised multi-operand epilogue (dummy-add constants)
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/levels.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_parity.log 2>&1; echo parity=$? >> gpurun_out/status.txt
for args in "--fixture vgg16 --mode dimension --pop 8 --prec bf16" "--fixture vgg16 --mode dimension --pop 8 --prec fp32" "--fixture resnet18 --mode dimension --pop 32 --prec fp32"; do
  echo "== $args" >> gpurun_out/levels.txt
  timeout 300 python scripts/conv_levels.py $args --order >> gpurun_out/levels.txt 2>&1
done
timeout 900 python -c "
import json, sys
sys.argv=['bench.py']
import bench
a = bench.parse()
peaks = json.load(open('MEASURED_PEAKS.json')) if __import__('os').path.exists('MEASURED_PEAKS.json') else {}
print(json.dumps(bench.workload_cfg4(a, peaks)))
" > gpurun_out/cfg4.json 2> gpurun_out/cfg4.err; echo cfg4=$? >> gpurun_out/status.txt
