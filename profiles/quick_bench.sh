# correctness spot checks + bench value for a list of configs
for a in "1 77 41" "1 481 65" "1 1920 1080" "2 77 41" "2 3840 2160" "2 1 1"; do timeout 120 python profiles/one_cfg.py $a 2>&1 | tail -1; done
for c in ${CFGS:-1 2}; do
python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('cfg', $c, round(d['value']), d['roofline'] and d['roofline']['kernel_ms'], d['roofline'] and d['roofline']['frac'], d['checked_vs_oracle'], d['clocks']['sm_mhz'])"
done
