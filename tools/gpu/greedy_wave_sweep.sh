for w in 1024 2048 4096 8192; do echo "wave=$w"; OPTS="{'wave': $w}" python tools/solve_timing.py 3 | tail -1 | cut -c1-160; done
for w in 64 148 296 592; do echo "wave=$w"; OPTS="{'wave': $w}" python tools/solve_timing.py 4 5 | cut -c1-160; done
for g in 1 4 8 16 32; do echo "group=$g"; SATURN_LS_GROUP=$g python tools/solve_timing.py 4 | cut -c1-160; done
