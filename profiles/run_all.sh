python -m pytest tests -q -m gpu -x > gpurun_out/pytest_s0.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_s0.log
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc $?"; cat gpurun_out/bench_default.json
for c in 1 3 4 5; do python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c$c.json 2>gpurun_out/bench_c$c.err; echo "cfg $c rc $?"; python -c "import json; d=json.load(open('gpurun_out/bench_c$c.json')); print($c, round(d['value']), d['roofline']['frac'], d['e2e']['value'] if d.get('e2e') else None, d['clocks']['sm_mhz'], d.get('checked_vs_oracle'))"; done
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>&1; echo "ref rc $?"; tail -1 gpurun_out/bench_ref.json
