# round 2 session 2: bisect the rare wrong forward: the round's pre-session tip (a93b375), TMA off, input im2col off
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/stress.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
echo "== a93b375" >> gpurun_out/stress.txt; (cd scratch/a93 && timeout 900 python scripts/stress_records.py 24) >> gpurun_out/stress.txt 2>&1
echo "== tma off" >> gpurun_out/stress.txt; TOBF_CONV_TMA=0 timeout 900 python scripts/stress_records.py 24 >> gpurun_out/stress.txt 2>&1
echo "== im2col off" >> gpurun_out/stress.txt; TOBF_INPUT_IM2COL=0 timeout 900 python scripts/stress_records.py 24 >> gpurun_out/stress.txt 2>&1
