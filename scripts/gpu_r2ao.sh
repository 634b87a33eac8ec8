# round 2 session 2: VGG-16 bf16 population (cfg4) with diagnostic builds: no drain/epilogue, no residual loads
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/variants.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in base nod noldg nostg; do
  lib=scripts/_probe_libs/libtobf_$v.so; [ $v = base ] && lib=paper_2107_09789_b200/libtobf.so
  TOBF_LIB=$lib timeout 600 python scripts/conv_levels.py --fixture vgg16 --mode dimension --pop 32 --prec bf16 > gpurun_out/vgg_levels_$v.txt 2>&1
  echo "== $v $(grep 'conv launches' gpurun_out/vgg_levels_$v.txt)" >> gpurun_out/variants.txt
done
