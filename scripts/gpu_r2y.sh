# round 2, call Y/Z: conv staging depth / shared-memory footprint variants (levels totals, A/B alternating)
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/variants.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rep in 1 2; do
for v in base sd6 sd7 ck8; do
  for prec in fp32 bf16; do
    echo "== $v $prec rep$rep $(TOBF_LIB=scripts/_probe_libs/libtobf_$v.so timeout 300 python scripts/conv_levels.py --prec $prec 2>&1 | grep 'conv launches')" >> gpurun_out/variants.txt
  done
done
done
echo done=0 >> gpurun_out/status.txt
