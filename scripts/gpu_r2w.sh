# round 2, call W: pipelined e2e (evaluate_stream, stream-ordered readbacks) — parity + bench e2e
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "stream or micro or population or eviction or smoke" > gpurun_out/pytest_stream.log 2>&1; echo stream=$? >> gpurun_out/status.txt
timeout 600 python bench.py --steps 20 --warmup 3 --no-sweeps --cfg4-pop 0 --gen-pop 0 --no-cpu-baseline > gpurun_out/bench_w.json 2> gpurun_out/bench_w.err; echo bench=$? >> gpurun_out/status.txt
timeout 600 python bench.py --steps 20 --warmup 3 --no-sweeps --cfg4-pop 0 --gen-pop 0 --no-cpu-baseline --e2e-depth 3 > gpurun_out/bench_w3.json 2> gpurun_out/bench_w3.err; echo bench3=$? >> gpurun_out/status.txt
