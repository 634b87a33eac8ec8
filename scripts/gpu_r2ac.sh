# round 2 (session 2): GPU suite at the tip + fresh per-role conv timings (TOBF_CONV_PROF) + levels
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status.txt
timeout 300 python scripts/conv_levels.py --prec fp32 > gpurun_out/levels_fp32.txt 2>&1; echo levels=$? >> gpurun_out/status.txt
TOBF_LIB=scripts/_probe_libs/libtobf_prof.so timeout 300 python scripts/conv_roles.py 0,1,2,3,4,14,20,22,29,34,38 > gpurun_out/roles.txt 2>&1; echo roles=$? >> gpurun_out/status.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/status.txt
