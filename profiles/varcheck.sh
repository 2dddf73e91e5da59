# correctness spot checks + device bench of variants/<name>/libgvx_cuda.so against the in-tree library
# usage: CHECKS="1 1920 1080;1 77 41" CFGS="1 5" bash profiles/varcheck.sh base name1 ...
L=paper_2008_11476_b200/lib/libgvx_cuda.so
cp $L /tmp/base.so
IFS=';' read -ra CHK <<< "${CHECKS:-3 7680 4320}"
for v in "$@"; do
  if [ $v != base ]; then cp variants/$v/libgvx_cuda.so $L; else cp /tmp/base.so $L; fi
  echo "== $v"
  for a in "${CHK[@]}"; do timeout 60 python profiles/diff_cfg.py $a 2>&1 | grep -v "^ rows\|^ cols\|^ [0-9]\|gpu s"; done
  for c in ${CFGS:-3}; do
  timeout 90 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --e2e-frames 0 --clock-window 0 --no-check 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('bench cfg', $c, round(d['value']), d['roofline']['frac'])"
  done
done
cp /tmp/base.so $L
