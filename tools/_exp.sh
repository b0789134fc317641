for it in 1 6; do timeout 300 python tools/join_round_time.py c4 1.0 $it 2>&1 | tail -1; done
timeout 300 python tools/join_round_time.py c1 1.0 10 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q -k "parity or golden or reference_suite or random" 2>&1 | tail -3
