for n in 513 700 1000 1100; do NGD_DEBUG_SYNC=1 PYTHONPATH=. timeout 300 python tools/chol_blocked_repro.py $n 2>&1 | tail -1; done
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -30
