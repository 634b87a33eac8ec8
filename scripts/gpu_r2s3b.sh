# round 2 session 3, call B: A-producer row prefetch (TOBF_CONV_APF 1 vs 0) A/B, race probe, conv parity
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/ab_*.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash scripts/build_variant_lib.sh apf0 -DTOBF_CONV_APF=0 > gpurun_out/variant.log 2>&1
for r in 1 2; do
  for v in tip apf0; do
    lib=""; [ $v = apf0 ] && lib="TOBF_LIB=scripts/_probe_libs/libtobf_apf0.so"
    env $lib timeout 300 python scripts/conv_levels.py > gpurun_out/ab_${v}_fp32_$r.txt 2>&1
    env $lib timeout 300 python scripts/conv_levels.py --prec bf16 > gpurun_out/ab_${v}_bf16_$r.txt 2>&1
  done
done
grep -h "conv launches" gpurun_out/ab_*.txt > /dev/null; for f in gpurun_out/ab_*.txt; do echo "$f $(head -1 $f)"; done > gpurun_out/ab_summary.txt
timeout 600 python scripts/race_probe.py 16 > gpurun_out/race_apf.txt 2>&1; echo race=$? >> gpurun_out/status.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo parity=$? >> gpurun_out/status.txt
