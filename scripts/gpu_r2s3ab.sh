# round 2 session 3, call AB: all-TMA variant without any gather code (issue() test made constant); levels, parity, race
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/ab_*.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for r in 1 2; do
  timeout 300 python scripts/conv_levels.py > gpurun_out/ab_tip_fp32_$r.txt 2>&1
  timeout 300 python scripts/conv_levels.py --prec bf16 > gpurun_out/ab_tip_bf16_$r.txt 2>&1
  TOBF_CONV_TMA_ALL=0 timeout 300 python scripts/conv_levels.py > gpurun_out/ab_mixed_fp32_$r.txt 2>&1
done
for f in gpurun_out/ab_*.txt; do echo "$f $(head -1 $f)"; done > gpurun_out/ab_summary.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo parity=$? >> gpurun_out/status.txt
timeout 600 python scripts/race_probe.py 12 > gpurun_out/race_fp32.txt 2>&1; echo race=$? >> gpurun_out/status.txt
