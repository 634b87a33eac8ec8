# round 2 session 3, call Z: split-K also in groups of up to 4 / 8 tiles per SM (TOBF_SPLIT_TILES_PER_SM 2 vs 4 vs 8); parity
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/ab_*.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash scripts/build_variant_lib.sh sp4 -DTOBF_SPLIT_TILES_PER_SM=4 > gpurun_out/variant.log 2>&1
bash scripts/build_variant_lib.sh sp8 -DTOBF_SPLIT_TILES_PER_SM=8 >> gpurun_out/variant.log 2>&1
for r in 1 2; do
  for v in tip sp4 sp8; do
    lib=""; [ $v != tip ] && lib="TOBF_LIB=scripts/_probe_libs/libtobf_$v.so"
    env $lib timeout 300 python scripts/conv_levels.py > gpurun_out/ab_${v}_fp32_$r.txt 2>&1
    env $lib timeout 300 python scripts/conv_levels.py --prec bf16 > gpurun_out/ab_${v}_bf16_$r.txt 2>&1
  done
done
for f in gpurun_out/ab_*.txt; do echo "$f $(head -1 $f)"; done > gpurun_out/ab_summary.txt
TOBF_LIB=scripts/_probe_libs/libtobf_sp4.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo parity=$? >> gpurun_out/status.txt
