# one build -> measure iteration on the GPU box: tests, bench line, ncu of one kernel
# usage: bash profiles/run_iter.sh <config> <kernel-regex> <tag>
CFG=${1:-2}; K=${2:-harris_kernel}; TAG=${3:-iter}
python -m pytest tests -q -m gpu -x > gpurun_out/pytest_$TAG.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_$TAG.log
python bench.py --config $CFG --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc $?"
python -c "import json; d=json.load(open('gpurun_out/bench_$TAG.json')); print('value', round(d['value']), 'ms', d['ms_per_step'], 'roof', d['roofline'], 'e2e', round(d['e2e']['value']), 'clk', d['clocks'], 'chk', d['checked_vs_oracle'])"
B="python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline --no-check --e2e-frames 1 --clock-window 0"
$B > gpurun_out/plain_$TAG.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/prof_$TAG $B > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu rc $?"
