for it in 1 6; do python tools/_exp.py c4 1.0 $it 2>&1 | tail -1; done
python tools/_exp.py c1 1.0 10 2>&1 | tail -1
python -m pytest tests -m gpu -x -q -k "parity or golden or reference_suite or random" 2>&1 | tail -3
