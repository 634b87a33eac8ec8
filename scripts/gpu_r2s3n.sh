# round 2 session 3, call N: A staging depth / TMEM A stages at BN=64 with the new A loop (A/B)
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/ab_*.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash scripts/build_variant_lib.sh sd3 -DTOBF_CONV_SD64=3 > gpurun_out/variant.log 2>&1
bash scripts/build_variant_lib.sh sd5 -DTOBF_CONV_SD64=5 -DTOBF_CONV_SD128=5 >> gpurun_out/variant.log 2>&1
bash scripts/build_variant_lib.sh sd6 -DTOBF_CONV_SD64=6 >> gpurun_out/variant.log 2>&1
for r in 1 2; do
  for v in tip sd3 sd5 sd6; do
    lib=""; [ $v != tip ] && lib="TOBF_LIB=scripts/_probe_libs/libtobf_$v.so"
    env $lib timeout 300 python scripts/conv_levels.py > gpurun_out/ab_${v}_fp32_$r.txt 2>&1
    env $lib timeout 300 python scripts/conv_levels.py --prec bf16 > gpurun_out/ab_${v}_bf16_$r.txt 2>&1
  done
done
for f in gpurun_out/ab_*.txt; do echo "$f $(head -1 $f)"; done > gpurun_out/ab_summary.txt
