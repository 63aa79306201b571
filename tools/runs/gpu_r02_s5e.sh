for m in plain sync nopdl plain; do timeout 300 python tools/ws_repro.py $m 2>&1 | tail -8; done
