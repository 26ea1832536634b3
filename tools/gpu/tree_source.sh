# k_tree<8> (config 1 full scan) SASS source page with per-instruction counts and stall samples.
python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/tree_plain.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tree -c 1 -o gpurun_out/tree_cfg1 \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_tree.log 2>&1
python tools/ncu_summary.py full gpurun_out/tree_cfg1.ncu-rep gpurun_out/r02l_ncu_full_k_tree_cfg1.json "r02l: k_tree<8> full scan, config 1" > /dev/null 2>&1
ncu -i gpurun_out/tree_cfg1.ncu-rep --page source --csv > gpurun_out/tree_cfg1_source.csv 2>/dev/null
ncu -i gpurun_out/tree_cfg1.ncu-rep --page details > gpurun_out/tree_cfg1_details.txt 2>/dev/null
rm -f gpurun_out/tree_cfg1.ncu-rep
ls -la gpurun_out | tail -5
