# round 2 session 2: where the streamed e2e blocks (host-call wall times), im2col on/off
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in 1 0 1; do
  TOBF_INPUT_IM2COL=$v timeout 600 python scripts/e2e_stall_probe.py 12 >> gpurun_out/e2e_stall.txt 2>&1; echo probe_x$v=$? >> gpurun_out/status.txt
done
