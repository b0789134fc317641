F="--no-cpu --no-recall --configs= --no-bf --no-c5 --no-rho-half --steps 5 --warmup 3"
python bench.py $F > gpurun_out/c2_new.json 2> gpurun_out/c2_new.err
python - <<PY
import json
d=json.loads(open('gpurun_out/c2_new.json').read().strip().splitlines()[-1])
print('c2 ms',d['ms_per_step'],d['phases_ms_per_step'],'apply',d['kernels']['apply']['ms_per_step'])
PY
python -m pytest tests -m gpu -x -q -k "parity or golden or random" 2>&1 | tail -3
