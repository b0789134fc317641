set -x
F="--steps 1 --warmup 1 --no-cpu --no-recall --configs= --no-bf --no-c5 --no-rho-half"
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_c2.csv python bench.py $F > gpurun_out/ncu_launch.log 2>&1
tail -n 2 gpurun_out/ncu_launch.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off -k regex:'k_join_mma|k_apply_stream|k_assemble' --csv --log-file gpurun_out/traffic_c2.csv python bench.py $F > gpurun_out/ncu_traffic.log 2>&1
tail -n 2 gpurun_out/ncu_traffic.log
python tools/full_parity.py c3 c4 c2 > gpurun_out/full_parity_final.json 2> gpurun_out/full_parity_final.err
tail -c 300 gpurun_out/full_parity_final.json
