# round 2 session 3, call AA: end-of-session check of the final tip — smoke, GPU suite, bench
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? >> gpurun_out/status.txt
