# round 2, call D: cfg2 full-size (rounding-decided verdict criterion), conv level timings fp32 vs bf16, ncu of a bf16 level
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -k cfg2 -s > gpurun_out/pytest_cfg2.log 2>&1; echo cfg2=$? >> gpurun_out/status.txt
for args in "--prec fp32" "--prec bf16" "--fixture vgg16 --mode dimension --pop 8 --prec fp32" "--fixture vgg16 --mode dimension --pop 8 --prec bf16"; do
  echo "== $args" >> gpurun_out/levels.txt
  timeout 300 python scripts/conv_levels.py $args --order >> gpurun_out/levels.txt 2>&1
done
echo levels=$? >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel --launch-skip 24 -c 1 -o gpurun_out/vgg_bf16_conv python scripts/conv_levels.py --fixture vgg16 --mode dimension --pop 8 --prec bf16 > gpurun_out/ncu_bf16.log 2>&1; echo ncu=$? >> gpurun_out/status.txt
