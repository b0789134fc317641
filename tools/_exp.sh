python -m pytest tests -m gpu -x -q -k "tc or lazy or parity or golden" 2>&1 | tail -4
F="--no-cpu --no-recall --no-bf --no-c5 --no-rho-half --steps 3 --warmup 2"
python bench.py $F --configs=c3 > gpurun_out/c3_new.json 2> gpurun_out/c3_new.err
python - <<PY
import json
d=json.loads(open('gpurun_out/c3_new.json').read().strip().splitlines()[-1])
c=d['configs']['c3']
print('c3 merge_s',c['merge_seconds'],c['phases_ms_per_step'])
PY
python tools/_exp.py c3 0.3 1 2>&1 | tail -1
