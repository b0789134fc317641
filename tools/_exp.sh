python -m pytest tests -m gpu -x -q 2>&1 | tail -3
F="--no-cpu --no-recall --no-bf --no-rho-half --steps 3 --warmup 2 --configs="
python bench.py $F > gpurun_out/c5_new.json 2> gpurun_out/c5_new.err
python - <<PY
import json
d=json.loads(open('gpurun_out/c5_new.json').read().strip().splitlines()[-1])
print('c2 ms',d['ms_per_step'],'c5',d['config5'])
PY
