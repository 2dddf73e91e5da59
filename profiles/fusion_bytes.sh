# DRAM bytes per output pixel before (run_naive, per-node kernels) and after
# fusion (run_plan program), every kernel of 2 executions under ncu (cold L2
# per kernel: each node's own traffic).  Frames per config: 265 Mpx per execution
# (inputs 2x L2, outputs and intermediates larger still, so writes leave L2 inside the kernel).
set -x
for spec in "1 128" "2 32" "3 8" "4 32"; do
  set -- $spec
  for nv in 1 0; do
    python profiles/fusion_session.py $1 $nv $2 > gpurun_out/fs_$1_$nv.log 2>&1 && \
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
        --log-file gpurun_out/fusion_$1_$nv.csv python profiles/fusion_session.py $1 $nv $2 > /dev/null 2>&1
    echo "cfg $1 naive $nv rc $?"
  done
done
