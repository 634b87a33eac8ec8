# round 2 session 3, call J: scheduler slot wait without backoff, 8-slot tile-info ring (A/B)
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/ab_*.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash scripts/build_variant_lib.sh nb -DTOBF_SCHED_NOBACKOFF > gpurun_out/variant.log 2>&1
bash scripts/build_variant_lib.sh i8 -DTOBF_CONV_INFO_SLOTS=8 >> gpurun_out/variant.log 2>&1
bash scripts/build_variant_lib.sh nbi8 -DTOBF_SCHED_NOBACKOFF -DTOBF_CONV_INFO_SLOTS=8 >> gpurun_out/variant.log 2>&1
for r in 1 2; do
  for v in tip nb i8 nbi8; do
    lib=""; [ $v != tip ] && lib="TOBF_LIB=scripts/_probe_libs/libtobf_$v.so"
    env $lib timeout 300 python scripts/conv_levels.py > gpurun_out/ab_${v}_fp32_$r.txt 2>&1
    env $lib timeout 300 python scripts/conv_levels.py --prec bf16 > gpurun_out/ab_${v}_bf16_$r.txt 2>&1
  done
done
for f in gpurun_out/ab_*.txt; do echo "$f $(head -1 $f)"; done > gpurun_out/ab_summary.txt
