# round 2, call C: bf16 + drop-in + full-size suites, cfg4 bf16 workload alone
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dropin.py -q --durations=10 > gpurun_out/pytest_parity.log 2>&1; echo parity=$? >> gpurun_out/status.txt
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q --durations=0 -k "cfg2 or bf16" > gpurun_out/pytest_full.log 2>&1; echo full=$? >> gpurun_out/status.txt
timeout 900 python -c "
import json, sys, argparse
sys.argv=['bench.py']
import bench
a = bench.parse()
peaks = json.load(open('MEASURED_PEAKS.json')) if __import__('os').path.exists('MEASURED_PEAKS.json') else {}
print(json.dumps(bench.workload_cfg4(a, peaks)))
" > gpurun_out/cfg4.json 2> gpurun_out/cfg4.err; echo cfg4=$? >> gpurun_out/status.txt
