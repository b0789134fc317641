python -m pytest tests -m gpu -x -q 2>&1 | tail -3
F="--no-cpu --no-recall --configs= --no-bf --no-c5 --no-rho-half --steps 5 --warmup 3"
python bench.py $F > gpurun_out/c2_new.json 2> gpurun_out/c2_new.err
python - <<PY
import json
d=json.loads(open('gpurun_out/c2_new.json').read().strip().splitlines()[-1])
print('c2 ms',d['ms_per_step'],'e2e',d['e2e'])
PY
