# round 2 session 3, call S: full-tile epilogue fast paths on the VGG-16 bf16 dimension population (cfg4 levels) and RN18; parity incl. dimension tests
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/ab_*.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash scripts/build_variant_lib.sh ef0 -DTOBF_EPI_FULL=0 > gpurun_out/variant.log 2>&1
for r in 1 2; do
  for v in tip ef0; do
    lib=""; [ $v != tip ] && lib="TOBF_LIB=scripts/_probe_libs/libtobf_$v.so"
    env $lib timeout 600 python scripts/conv_levels.py --fixture vgg16 --mode dimension --pop 32 --prec bf16 > gpurun_out/ab_${v}_vgg_$r.txt 2>&1
  done
done
for f in gpurun_out/ab_*.txt; do echo "$f $(head -1 $f)"; done > gpurun_out/ab_summary.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dimattack.py tests/test_gpu_fullsize.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo parity=$? >> gpurun_out/status.txt
timeout 900 python scripts/race_probe.py 6 --fixture vgg16 --mode dimension --pop 8 --prec bf16 > gpurun_out/race_vgg.txt 2>&1; echo racevgg=$? >> gpurun_out/status.txt
