# local search: warps per walker (SATURN_LS_GROUP) x config, time to the best plan
for k in 1 4 8; do
  echo "== SATURN_LS_GROUP=$k"
  SATURN_LS_GROUP=$k timeout 600 python tools/ls_wave_sweep.py 3 4 5 2>&1 | grep "wave=4096" | cut -c1-120
done
