# round 2 session 3, call F: per-role conv timings at the tip (prof build)
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash scripts/build_prof_lib.sh > gpurun_out/prof_build.log 2>&1
TOBF_LIB=scripts/_probe_libs/libtobf_prof.so timeout 300 python scripts/conv_roles.py 0,2,4,5,6,10,20,22,34,45,47 > gpurun_out/roles.txt 2>&1; echo roles=$? >> gpurun_out/status.txt
