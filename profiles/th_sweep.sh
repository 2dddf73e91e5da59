# device bench of one config at forced tile heights: CFG=1 VAR=GVX_EDGE_TH THS="40 36 32" bash profiles/th_sweep.sh
for th in ${THS}; do
  if [ $th = 0 ]; then unset $VAR; else export $VAR=$th; fi
  timeout 90 python bench.py --config $CFG --steps 20 --warmup 5 --no-cpu-baseline --e2e-frames 0 --clock-window 0 --no-check 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('cfg', $CFG, 'th', $th, round(d['value']), d['roofline']['frac'])"
done
