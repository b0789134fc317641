timeout 600 python tools/join_round_time.py c3 1.0 9 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q -k "tc_lazy or lazy or parity or golden" 2>&1 | tail -3
F="--no-cpu --no-recall --no-bf --no-c5 --no-rho-half --steps 3 --warmup 2"
python bench.py $F --configs=c3 > gpurun_out/c3_new.json 2> gpurun_out/c3_new.err
python - <<PY
import json
d=json.loads(open('gpurun_out/c3_new.json').read().strip().splitlines()[-1])
c=d['configs']['c3']
print('c3 merge_s',c['merge_seconds'],'exact',c['exact_evals_per_step'],c['kernels']['apply']['fp64']['lazy_batches_per_step'],c['phases_ms_per_step'])
PY
