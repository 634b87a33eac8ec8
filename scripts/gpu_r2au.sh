# round 2 session 2: bisect the headline-test mismatch: HEAD ops.cu vs current ops.cu (twice)
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
TOBF_LIB=scripts/_probe_libs/libtobf_opshead.so timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k headline > gpurun_out/pytest_opshead.log 2>&1; echo opshead=$? >> gpurun_out/status.txt
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k headline > gpurun_out/pytest_cur1.log 2>&1; echo cur1=$? >> gpurun_out/status.txt
