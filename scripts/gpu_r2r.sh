# round 2, call R: role timings of the TMA conv, rb8 LSTM ncu, e2e worker-count probe
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash scripts/build_prof_lib.sh > gpurun_out/prof_build.log 2>&1
TOBF_LIB=scripts/_probe_libs/libtobf_prof.so timeout 300 python scripts/conv_roles.py 0,1,3,4,20,34,38 > gpurun_out/roles.txt 2>&1; echo roles=$? >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lstm_ctc_rb --launch-skip 1 -c 1 -o gpurun_out/lstm512_rb8 python scripts/cfg5_lstm.py --hidden 512 --reps 1 > gpurun_out/ncu_lstm.log 2>&1; echo ncul8=$? >> gpurun_out/status.txt
for w in 14 15; do echo "== workers $w" >> gpurun_out/e2e_workers.txt; TOBF_HOST_WORKERS=$w timeout 300 python scripts/e2e_timeline.py 32 2>&1 | grep -E "total|device" >> gpurun_out/e2e_workers.txt; done
