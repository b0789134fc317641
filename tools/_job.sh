set -x
python tools/full_parity.py c3 c4 c2 > gpurun_out/full_parity_r2b.json 2> gpurun_out/full_parity_r2b.err
tail -c 600 gpurun_out/full_parity_r2b.json
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_join_tc -c 1 -o gpurun_out/c3_tc -f python tools/profile_config.py c3 --scale 0.3 > gpurun_out/ncu_c3.log 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_join_dense -c 1 -o gpurun_out/c4_dense -f python tools/profile_config.py c4 --scale 0.3 > gpurun_out/ncu_c4.log 2>&1
tail -3 gpurun_out/ncu_c3.log gpurun_out/ncu_c4.log
