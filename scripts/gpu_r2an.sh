# round 2 session 2: VGG-16 bf16 population levels (cfg4), input im2col on/off
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in 1 0; do
  TOBF_INPUT_IM2COL=$v timeout 600 python scripts/conv_levels.py --fixture vgg16 --mode dimension --pop 32 --prec bf16 > gpurun_out/vgg_levels_x$v.txt 2>&1; echo vgg_x$v=$? >> gpurun_out/status.txt
done
