# Block-pass (block.cuh) configurations of the d = 6 chains under ncu launch
# timing: groups G, slots NB and row width R (32-a blocks) per run, e.g.
#   bash tools/block_cfg_runs.sh "4 4 32" "2 3 32" "2 2 32"
# (MUMODE_BLOCK_G / _NB / _R override the planner's choice; results in gpurun_out/)
for cfg in "$@"; do set -- $cfg; for n in 18 20; do
  MUMODE_BLOCK_G=$1 MUMODE_BLOCK_NB=$2 MUMODE_BLOCK_R=$3 MUMODE_BLOCK_DEBUG=1 timeout 120 \
    ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof.py d6 $n --policy 16 \
    > gpurun_out/blkcfg_${n}_${1}_${2}_$3.csv 2>&1
  python tools/ktimes.py gpurun_out/blkcfg_${n}_${1}_${2}_$3.csv 4
done; done
