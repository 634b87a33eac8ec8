# round 2 session 3, call E: raw-hi tf32 split (TOBF_CONV_RAWHI) x fp32 row prefetch A/B; parity
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/ab_*.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash scripts/build_variant_lib.sh raw -DTOBF_CONV_APF_F32=0 > gpurun_out/variant.log 2>&1
bash scripts/build_variant_lib.sh orig -DTOBF_CONV_APF_F32=0 -DTOBF_CONV_RAWHI=0 >> gpurun_out/variant.log 2>&1
for r in 1 2; do
  for v in tip raw orig; do
    lib=""; [ $v != tip ] && lib="TOBF_LIB=scripts/_probe_libs/libtobf_$v.so"
    env $lib timeout 300 python scripts/conv_levels.py > gpurun_out/ab_${v}_fp32_$r.txt 2>&1
  done
done
for f in gpurun_out/ab_*.txt; do echo "$f $(head -1 $f)"; done > gpurun_out/ab_summary.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo parity=$? >> gpurun_out/status.txt
TOBF_LIB=scripts/_probe_libs/libtobf_raw.so timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_parity_raw.log 2>&1; echo parityraw=$? >> gpurun_out/status.txt
