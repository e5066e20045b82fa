# block-pass configurations under ncu launch timing: G NB R per run
for cfg in "2 2 32" "1 2 32" "4 6 16"; do set -- $cfg; for n in 18 20; do
  MUMODE_BLOCK_WIDE=1 MUMODE_BLOCK_R=$3 MUMODE_BLOCK_NB=$2 MUMODE_BLOCK_G=$1 MUMODE_BLOCK_DEBUG=1 timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof.py d6 $n --policy 16 > gpurun_out/w_${n}_${1}_${2}_$3.csv 2>&1
done; done
