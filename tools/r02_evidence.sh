# Round-2 evidence run (one B200): bench launch list, ncu --set full of the
# headline C2 mode kernel and of the 18^6 chain (cube + pair + skinny), parity
# report against the reference library.
set -x
ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/r02_launches.csv 2> gpurun_out/r02_launches.err
ncu --set full --clock-control none --import-source on -k regex:modeprod_tma -s 3 -c 1 -o gpurun_out/r02_c2 python tools/prof.py c2 > gpurun_out/r02_c2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"block_kernel|skinny" -s 3 -c 3 -o gpurun_out/r02_d6_18 python tools/prof.py d6 18 > gpurun_out/r02_d6_18.log 2>&1
timeout 900 python tools/parity_report.py > gpurun_out/r02_parity.json 2> gpurun_out/r02_parity.err
