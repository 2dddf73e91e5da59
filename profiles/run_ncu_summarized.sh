# run_ncu.sh, then summarise each capture on the box and drop the reports
# (gpurun copies back at most 64 MiB): profiles/ncu_<TAG>.json + ncu_traffic.json
set -x
bash profiles/run_ncu.sh > gpurun_out/run_ncu.log 2>&1
reps=$(ls gpurun_out/prof_cfg*.ncu-rep 2>/dev/null)
python profiles/summarize_ncu.py ${TAG:-r2d} $reps > gpurun_out/summary.log 2>&1
cp profiles/ncu_${TAG:-r2d}.json profiles/ncu_traffic.json gpurun_out/
for r in $reps; do
  ncu -i $r --page source --csv --print-source sass > ${r%.ncu-rep}.src.csv 2>/dev/null
  python profiles/sass_hot.py ${r%.ncu-rep}.src.csv > ${r%.ncu-rep}.sass.txt 2>/dev/null
  rm -f ${r%.ncu-rep}.src.csv $r
done
