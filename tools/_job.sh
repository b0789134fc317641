set -x
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; tail -n 3 gpurun_out/gputest.log
python tools/full_parity.py c3 > gpurun_out/full_parity_c3.json 2> gpurun_out/full_parity_c3.err
tail -c 200 gpurun_out/full_parity_c3.json
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 200 gpurun_out/bench.json
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:k_join_tc -c 1 -o gpurun_out/c3_tc4 -f python tools/profile_config.py c3 --scale 0.3 > gpurun_out/ncu_c3.log 2>&1
tail -n 2 gpurun_out/ncu_c3.log
