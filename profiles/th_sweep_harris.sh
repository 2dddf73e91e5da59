for th in ${THS:-0 216 180 135 108 90 72}; do
  if [ $th = 0 ]; then unset GVX_HARRIS_TH; else export GVX_HARRIS_TH=$th; fi
  timeout 90 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline --e2e-frames 0 --clock-window 0 --no-check 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('th', $th, round(d['value']), d['roofline']['frac'])"
done
