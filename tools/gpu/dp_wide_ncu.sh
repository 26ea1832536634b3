# Wide state-space search: rates on a few multi-node workloads, and ncu of one large level.
for a in "14 3 4 114 15 25" "14 2 4 112 23 25" "14 2 8 113 15 23" "12 2 4 124 22 23 exact" "14 4 8 115 12 23"; do
  timeout 300 python tools/dp_wide_probe.py $a >> gpurun_out/dpw_rates.txt 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dp_expand_wide -s 9 -c 1 -o gpurun_out/dpw \
  python tools/dp_wide_probe.py 14 3 4 114 15 25 > gpurun_out/ncu_dpw.log 2>&1
python tools/ncu_summary.py full gpurun_out/dpw.ncu-rep gpurun_out/dpw_ncu.json "k_dp_expand_wide, J=14 3x4 GPUs seed 114 T=15, level 10" > /dev/null 2>&1
ncu -i gpurun_out/dpw.ncu-rep --page source --csv > gpurun_out/dpw_source.csv 2>/dev/null
ncu -i gpurun_out/dpw.ncu-rep --page details > gpurun_out/dpw_details.txt 2>/dev/null
rm -f gpurun_out/dpw.ncu-rep
cat gpurun_out/dpw_rates.txt
