# round 2 session 2: stress the headline records (resident + e2e) for wrong forwards: current, HEAD ops.cu, no input im2col
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/stress.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
echo "== current" >> gpurun_out/stress.txt; timeout 900 python scripts/stress_records.py 8 >> gpurun_out/stress.txt 2>&1
echo "== opshead" >> gpurun_out/stress.txt; TOBF_LIB=scripts/_probe_libs/libtobf_opshead.so timeout 900 python scripts/stress_records.py 8 >> gpurun_out/stress.txt 2>&1
echo "== no input im2col" >> gpurun_out/stress.txt; TOBF_INPUT_IM2COL=0 timeout 900 python scripts/stress_records.py 8 >> gpurun_out/stress.txt 2>&1
