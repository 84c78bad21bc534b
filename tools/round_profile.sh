# Round-end evidence on one GPU: launch list (device time per kernel), per-kernel DRAM traffic
# (-> profiles/ncu_traffic.json), one full ncu capture of the top kernel.  CONFIG (default glm9b)
C=${CONFIG:-glm9b}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$C.csv \
    python bench.py --config $C --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/launches_$C.log 2>&1
python tools/summarize_ncu_launches.py gpurun_out/launches_$C.csv --last-steps 1 > gpurun_out/launches_${C}_summary.txt
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/traffic_$C.csv \
    python bench.py --config $C --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/traffic_$C.log 2>&1
python tools/ncu_traffic.py gpurun_out/traffic_$C.csv $C
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
