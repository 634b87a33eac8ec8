# round 2, call B: parity suite (incl. bf16 mode), full-size suite, quick bench
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --durations=15 > gpurun_out/pytest_parity.log 2>&1; echo parity=$? >> gpurun_out/status.txt
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q --durations=0 > gpurun_out/pytest_full.log 2>&1; echo full=$? >> gpurun_out/status.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --gen-pop 0 --cfg4-pop 0 > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo bench=$? >> gpurun_out/status.txt
