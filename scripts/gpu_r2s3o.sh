# round 2 session 3, call O: tile-claim batch size / threshold A/B
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/ab_*.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash scripts/build_variant_lib.sh c2 -DTOBF_CONV_CLAIM=2 > gpurun_out/variant.log 2>&1
bash scripts/build_variant_lib.sh c8 -DTOBF_CONV_CLAIM=8 >> gpurun_out/variant.log 2>&1
bash scripts/build_variant_lib.sh m4 -DTOBF_CONV_CLAIM_MIN=4 >> gpurun_out/variant.log 2>&1
for r in 1 2; do
  for v in tip c2 c8 m4; do
    lib=""; [ $v != tip ] && lib="TOBF_LIB=scripts/_probe_libs/libtobf_$v.so"
    env $lib timeout 300 python scripts/conv_levels.py > gpurun_out/ab_${v}_fp32_$r.txt 2>&1
  done
done
for f in gpurun_out/ab_*.txt; do echo "$f $(head -1 $f)"; done > gpurun_out/ab_summary.txt
