# round 2 session 2: race localisation variants (E2: slot released after the split; E3: every drain warp waits on acc_full; TMA off)
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/race_*.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
TOBF_LIB=scripts/_probe_libs/libtobf_e2.so timeout 900 python scripts/race_probe.py 30 > gpurun_out/race_e2.txt 2>&1
TOBF_LIB=scripts/_probe_libs/libtobf_e3.so timeout 900 python scripts/race_probe.py 30 > gpurun_out/race_e3.txt 2>&1
TOBF_CONV_TMA=0 timeout 900 python scripts/race_probe.py 30 > gpurun_out/race_notma.txt 2>&1
timeout 900 python scripts/race_probe.py 30 > gpurun_out/race_base.txt 2>&1
