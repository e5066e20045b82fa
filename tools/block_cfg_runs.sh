for cfg in "2 3" "2 4" "4 4" "4 5" "4 6" "2 6"; do set -- $cfg; for n in 18 20 12 14; do
  MUMODE_BLOCK_NB=$2 MUMODE_BLOCK_G=$1 timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof.py d6 $n --policy 16 > gpurun_out/c_${n}_${1}_$2.csv 2>&1
done; done
