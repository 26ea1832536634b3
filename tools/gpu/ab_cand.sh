# A/B of a k_cand build variant on the sampled configs: bench lines alternating base / variant.
V=paper_2311_02840_b200/_lib/variants/$1.so
for rep in 1 2; do
  for c in 3 5; do
    python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('base cfg$c', '%.4g' % d['value'])"
    SATURN_ENGINE_LIB=$V python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$1 cfg$c', '%.4g' % d['value'])"
  done
done
