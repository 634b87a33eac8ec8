# round 2 session 2: full GPU suite with the race fix + tail alignment default, records stress, bench
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/stress.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
echo "== stress" >> gpurun_out/stress.txt; timeout 900 python scripts/stress_records.py 24 >> gpurun_out/stress.txt 2>&1
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? >> gpurun_out/status.txt
