# round 2 session 2: determinism probe on the other paths: bf16 headline, VGG-16 dimension bf16 and fp32
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/race_*.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python scripts/race_probe.py 20 --prec bf16 > gpurun_out/race_bf16.txt 2>&1; echo bf16=$? >> gpurun_out/status.txt
timeout 1200 python scripts/race_probe.py 8 --fixture vgg16 --mode dimension --pop 8 --prec bf16 > gpurun_out/race_vgg_bf16.txt 2>&1; echo vggbf16=$? >> gpurun_out/status.txt
timeout 1200 python scripts/race_probe.py 8 --fixture vgg16 --mode dimension --pop 8 > gpurun_out/race_vgg_fp32.txt 2>&1; echo vggfp32=$? >> gpurun_out/status.txt
