# round 2 session 2: correction accumulator drained before the tile's last main chunk (TOBF_CORR_FIRST) A/B
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/variants.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "conv or execute" > gpurun_out/pytest_conv.log 2>&1; echo pytest_conv=$? >> gpurun_out/status.txt
for rep in 1 2; do
  for v in new cf0; do
    lib=scripts/_probe_libs/libtobf_$v.so; [ $v = new ] && lib=paper_2107_09789_b200/libtobf.so
    TOBF_LIB=$lib timeout 300 python scripts/conv_levels.py --prec fp32 > gpurun_out/levels_${v}_$rep.txt 2>&1
    echo "== $v rep$rep $(grep 'conv launches' gpurun_out/levels_${v}_$rep.txt)" >> gpurun_out/variants.txt
  done
done
