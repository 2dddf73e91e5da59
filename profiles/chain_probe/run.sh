# ncu kernel lists of one 4K corpus graph with and without the opt-in
# generic local -> local chains (GVX_LOCAL_CHAINS=1)
for f in sobel_4k edge_fig1_4k; do
  for mode in chain nochain; do
    if [ $mode = chain ]; then export GVX_LOCAL_CHAINS=1; else unset GVX_LOCAL_CHAINS; fi
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
        --log-file gpurun_out/chain_${f}_${mode}.csv python profiles/chain_probe/run.py profiles/chain_probe/$f.json \
        > gpurun_out/chain_${f}_${mode}.log 2>&1
    echo "$f $mode rc $?"
  done
done
