# round 2 session 3, call D: fp32 A-row prefetch after the TMEM stores (TOBF_CONV_APF_F32 1 vs 0), race probes
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/ab_*.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash scripts/build_variant_lib.sh f0 -DTOBF_CONV_APF_F32=0 > gpurun_out/variant.log 2>&1
for r in 1 2 3; do
  for v in tip f0; do
    lib=""; [ $v = f0 ] && lib="TOBF_LIB=scripts/_probe_libs/libtobf_f0.so"
    env $lib timeout 300 python scripts/conv_levels.py > gpurun_out/ab_${v}_fp32_$r.txt 2>&1
  done
done
for f in gpurun_out/ab_*.txt; do echo "$f $(head -1 $f)"; done > gpurun_out/ab_summary.txt
timeout 600 python scripts/race_probe.py 12 > gpurun_out/race_fp32.txt 2>&1; echo race=$? >> gpurun_out/status.txt
timeout 600 python scripts/race_probe.py 12 --prec bf16 > gpurun_out/race_bf16.txt 2>&1; echo raceb=$? >> gpurun_out/status.txt
