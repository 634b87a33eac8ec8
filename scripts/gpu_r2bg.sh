# round 2 session 2: stem pairing (two candidates' stems as one 128-channel problem): parity, race probe, levels A/B
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt gpurun_out/variants.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/status.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo parity=$? >> gpurun_out/status.txt
timeout 900 python scripts/race_probe.py 20 > gpurun_out/race_pair.txt 2>&1; echo race=$? >> gpurun_out/status.txt
for rep in 1 2; do
  for v in 1 0; do
    for prec in fp32 bf16; do
      TOBF_PAIR_STEMS=$v timeout 300 python scripts/conv_levels.py --prec $prec > gpurun_out/levels_pair${v}_${prec}_$rep.txt 2>&1
      echo "== pair=$v $prec rep$rep $(grep 'conv launches' gpurun_out/levels_pair${v}_${prec}_$rep.txt)" >> gpurun_out/variants.txt
    done
  done
done
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "headline" > gpurun_out/pytest_full.log 2>&1; echo full=$? >> gpurun_out/status.txt
