# round 2, call F: conv role timings (prof build), e2e timeline at P=32, LER instruction count, racecheck
set -x
mkdir -p gpurun_out; rm -f gpurun_out/status.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
bash scripts/build_prof_lib.sh > gpurun_out/prof_build.log 2>&1
TOBF_LIB=scripts/_probe_libs/libtobf_prof.so timeout 300 python scripts/conv_roles.py 0,1,2,3,4,20,22,34,38 > gpurun_out/roles.txt 2>&1; echo roles=$? >> gpurun_out/status.txt
timeout 300 python scripts/e2e_timeline.py 32 > gpurun_out/timeline32.txt 2>&1; echo tl=$? >> gpurun_out/status.txt
timeout 300 python scripts/ler_instr.py > gpurun_out/ler_tokens.txt 2>&1
timeout 600 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum --clock-control none -k regex:levenshtein_bp -c 1 --csv --log-file gpurun_out/ler_instr.csv python scripts/ler_instr.py > gpurun_out/ncu_ler.log 2>&1; echo nculer=$? >> gpurun_out/status.txt
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard python -m pytest tests/test_gpu_parity.py -q -x -k "conv_kernel_matches_oracle and (case3 or case5)" > gpurun_out/racecheck.log 2>&1; echo race=$? >> gpurun_out/status.txt
