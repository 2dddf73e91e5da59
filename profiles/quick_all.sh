# GPU parity suite + device-only bench line of each config (no e2e leg, no CPU baseline)
# usage: [CFGS="1 2 3 4 5"] [NOTEST=1] bash profiles/quick_all.sh
if [ -z "$NOTEST" ]; then
python -m pytest tests -q -m gpu -x > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/pytest_quick.log
fi
for c in ${CFGS:-1 2 3 4 5}; do
python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --e2e-frames 0 --clock-window 0.5 2>gpurun_out/quick_c$c.err | python -c "import json,sys; d=json.load(sys.stdin); r=d['roofline']; print('cfg', $c, round(d['value']), r and r['kernel_ms'], r and r['frac'], 'chk', d['checked_vs_oracle'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/quick_c$c.err
done
