# round 2, call X: evaluate_stream with the next batch pre-dealt to the host workers
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "stream or micro" > gpurun_out/pytest_stream.log 2>&1; echo stream=$? >> gpurun_out/status.txt
B="python bench.py --steps 20 --warmup 3 --no-sweeps --cfg4-pop 0 --gen-pop 0 --no-cpu-baseline"
timeout 600 $B > gpurun_out/bench_x2.json 2> gpurun_out/bench_x2.err; echo b2=$? >> gpurun_out/status.txt
timeout 600 $B --micro 32 > gpurun_out/bench_x2m.json 2> gpurun_out/bench_x2m.err; echo b2m=$? >> gpurun_out/status.txt
timeout 600 $B --micro 32 --e2e-depth 3 > gpurun_out/bench_x3m.json 2> gpurun_out/bench_x3m.err; echo b3m=$? >> gpurun_out/status.txt
timeout 600 $B --micro 16 > gpurun_out/bench_x2m16.json 2> gpurun_out/bench_x2m16.err; echo b2m16=$? >> gpurun_out/status.txt
