# bench each variants/<name>/libgvx_cuda.so against the in-tree library (cfg $CFG)
# usage: CFG=2 bash profiles/run_variants.sh name1 name2 ...
CFG=${CFG:-2}
L=paper_2008_11476_b200/lib/libgvx_cuda.so
cp $L /tmp/base_libgvx_cuda.so
for v in base "$@" base; do
  if [ $v = base ]; then cp /tmp/base_libgvx_cuda.so $L; else cp variants/$v/libgvx_cuda.so $L; fi
  python bench.py --config $CFG --steps 20 --warmup 5 --no-cpu-baseline --e2e-frames 0 --clock-window 0.5 2>gpurun_out/var_$v.err | python -c "import json,sys; d=json.load(sys.stdin); print('$v', 'cfg', $CFG, round(d['value']), d['roofline']['kernel_ms'], d['roofline']['frac'], 'chk', d['checked_vs_oracle'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/var_$v.err
done
cp /tmp/base_libgvx_cuda.so $L
