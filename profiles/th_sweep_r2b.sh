B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-frames 0 --no-single --clock-window 0.5"
for c in 5 1; do for t in auto 24 32 48 64; do
  if [ $t = auto ]; then $B --config $c > /tmp/o.json 2>/dev/null; else GVX_EDGE8_TH=$t $B --config $c > /tmp/o.json 2>/dev/null; fi
  python -c "import json; d=json.load(open('/tmp/o.json')); print('cfg', $c, 'th', '$t', round(d['value']), d['roofline']['frac'], d['clocks']['sm_mhz'])"
done; done
for t in auto 16 24 32 48 64; do
  if [ $t = auto ]; then $B --config 2 > /tmp/o.json 2>/dev/null; else GVX_HARRIS_TH=$t $B --config 2 > /tmp/o.json 2>/dev/null; fi
  python -c "import json; d=json.load(open('/tmp/o.json')); print('cfg', 2, 'th', '$t', round(d['value']), d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
