# ncu DRAM traffic + duration of every kernel of two eager V(1,1) cycles, all five configs
mkdir -p gpurun_out
for c in c1 c2 c3 c4 c5; do
  python scripts/one_cycle.py $c > gpurun_out/traffic_$c.out 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/traffic_$c.csv python scripts/one_cycle.py $c > /dev/null 2>&1; echo $c=$?
done
