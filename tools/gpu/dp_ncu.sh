# ncu captures of the state-space kernels after the round-2 packing work: the widest one-node
# level of config 3's proof, and a wide homogeneous level (3 x 4 GPUs).
summ() {
  python tools/ncu_summary.py full gpurun_out/$1.ncu-rep gpurun_out/$2 "$3" > /dev/null 2>&1
  ncu -i gpurun_out/$1.ncu-rep --page details > gpurun_out/$1_details.txt 2>/dev/null
  rm -f gpurun_out/$1.ncu-rep
}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dp_expand -s 8 -c 1 -o gpurun_out/dp1 \
  python tools/dp_probe.py 3 29 > gpurun_out/ncu_dp1.log 2>&1
summ dp1 r02t_ncu_full_dp_expand_cfg3.json "r02t: k_dp_expand<8>, config 3 proof at T = 29, level 8 -> 9 (packed placement)"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dpw_expand_h -s 22 -c 1 -o gpurun_out/dpw \
  python tools/dp_wide_probe.py 14 3 4 114 15 25 > gpurun_out/ncu_dpw.log 2>&1
summ dpw r02t_ncu_full_dpw_expand_h_3x4.json "r02t: k_dpw_expand_h<3,4>, J=14 on 3 x 4 GPUs (seed 114), T=15, a 2.97 M-state level"
grep -E "Duration|Issue Slots Busy|Achieved Occ|Registers Per" gpurun_out/dp1_details.txt gpurun_out/dpw_details.txt
