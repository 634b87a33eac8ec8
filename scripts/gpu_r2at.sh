# round 2 session 2: isolate the e2e record mismatch: full-size headline test with tail alignment off / on
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
TOBF_TAIL_ALIGN=0 timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k headline > gpurun_out/pytest_f0.log 2>&1; echo f0=$? >> gpurun_out/status.txt
TOBF_TAIL_ALIGN=0.5 TOBF_HOST_WORKERS=0 timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k headline > gpurun_out/pytest_f5_w0.log 2>&1; echo f5w0=$? >> gpurun_out/status.txt
