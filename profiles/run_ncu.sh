# ncu --set full of each config's dominant kernel (after the same command
# ran clean without ncu), then the launch list of the cfg2 bench.
set -x
# --e2e-frames 0 skips the host pipeline leg; -s 3 skips the warm-up batch launches,
# so the capture is a full batch launch like the timed ones
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-check --e2e-frames 0 --clock-window 0"
for c in ${CFGS:-2 1 3 4}; do
  K=$(python -c "print({1:'edge8?_kernel',2:'harris4?_kernel',3:'sep_kernel',4:'sep_kernel',5:'edge8_kernel'}[$c])")
  $B --config $c > gpurun_out/plain_$c.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/prof_cfg$c $B --config $c > gpurun_out/ncu_$c.log 2>&1
  echo "cfg $c rc $?"
done
if [ -z "$NO_LAUNCHES" ]; then
LC=${LAUNCH_CFG:-5}
$B --config $LC > gpurun_out/plain_l.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_cfg$LC.csv $B --config $LC > /dev/null 2>&1; echo launches $?
fi
