# round 2 session 2: DRAM traffic of one bench step's conv launches (profiles/conv_traffic.json)
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --print-units base -k regex:conv_tc_kernel --launch-skip 54 -c 54 --csv --log-file gpurun_out/conv_traffic.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-sweeps --cfg4-pop 0 --gen-pop 0 > gpurun_out/ncu_traffic.log 2>&1; echo traffic=$? >> gpurun_out/status.txt
