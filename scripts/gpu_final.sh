# End-of-round verification: smoke, GPU tests, bench (+ reference arm), launch list of the
# headline step and an ncu full capture of the dimension-attacker kernel. Outputs in gpurun_out/.
set -x
rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? >> gpurun_out/status.txt
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$? >> gpurun_out/status.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-sweeps --cfg4-pop 0 --gen-pop 0 > gpurun_out/ncu_launch.log 2>&1; echo ncul=$? >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:forest_predict -c 1 -o gpurun_out/forest_full python -m pytest tests/test_gpu_dimattack.py -q -k kernel_vs_oracle > gpurun_out/ncu_forest.log 2>&1; echo ncuforest=$? >> gpurun_out/status.txt
