# round 2 session 3, call C: non-blocking A-row prefetch A/B (TOBF_CONV_APF), tf32 operand-rounding probe
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/ab_*.txt
nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -Ipaper_2107_09789_b200/csrc scripts/tf32_trunc_probe.cu -o /tmp/tp && /tmp/tp > gpurun_out/tf32_probe.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash scripts/build_variant_lib.sh apf0 -DTOBF_CONV_APF=0 > gpurun_out/variant.log 2>&1
for r in 1 2; do
  for v in tip apf0; do
    lib=""; [ $v = apf0 ] && lib="TOBF_LIB=scripts/_probe_libs/libtobf_apf0.so"
    env $lib timeout 300 python scripts/conv_levels.py > gpurun_out/ab_${v}_fp32_$r.txt 2>&1
    env $lib timeout 300 python scripts/conv_levels.py --prec bf16 > gpurun_out/ab_${v}_bf16_$r.txt 2>&1
  done
done
for f in gpurun_out/ab_*.txt; do echo "$f $(head -1 $f)"; done > gpurun_out/ab_summary.txt
timeout 600 python scripts/race_probe.py 16 > gpurun_out/race_apf.txt 2>&1; echo race=$? >> gpurun_out/status.txt
