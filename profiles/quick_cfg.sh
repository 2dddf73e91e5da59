# bench value / roofline / e2e for a list of configs (CFGS), no CPU leg
for c in ${CFGS:-3 4}; do
python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline'] or {}; print('cfg', $c, round(d['value']), r.get('frac'), r.get('kernel_ms'), round(d['e2e']['value']), d['checked_vs_oracle'], d['clocks']['sm_mhz'])"
done
