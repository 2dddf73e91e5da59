for f in sobel_4k edge_fig1_4k; do
  for env in "" "GVX_NO_LOCAL_CHAINS=1"; do
    env $env ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/chain_${f}_${env:+nochain}.csv python profiles/chain_probe/run.py profiles/chain_probe/$f.json > gpurun_out/chain_${f}_${env:+nochain}.log 2>&1
    echo "$f $env rc $?"
  done
done
