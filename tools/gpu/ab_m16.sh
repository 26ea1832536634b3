# A/B of k_cand / k_ls build variants at config 4 (Multi16 layout): bench line per variant,
# then the GPU suite against the first variant.  Usage: bash tools/gpu/ab_m16.sh v1 v2 ...
V=paper_2311_02840_b200/_lib/variants
for rep in 1 2; do
  python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_base_$rep.log 2>&1
  for v in "$@"; do
    SATURN_ENGINE_LIB=$V/$v.so python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_${v}_$rep.log 2>&1
  done
done
SATURN_ENGINE_LIB=$V/$1.so timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_tests_$1.log 2>&1; echo tests_exit=$? >> gpurun_out/ab_tests_$1.log
for f in gpurun_out/ab_*.log; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads([l for l in open(f) if l.startswith('{')][-1])
    t = d.get('time_to_best') or {}
    print(f, '%.4g' % d['value'], 'ttb_dev_ms %.3f' % (1e3 * (t.get('device_s') or 0)), 'wall_ms %.3f' % (1e3 * (t.get('wall_s') or 0)), t.get('status'))
except Exception as e:
    pass
PY
done
