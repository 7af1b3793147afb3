export PYTHONPATH=.
for p in 0 1; do CBB_TC_PAIR=$p timeout 100 python scripts/probe_mfk.py 2>&1 | tail -2 | sed "s/^/pair=$p /"; done
timeout 300 python -m pytest tests/test_gpu_projection.py -m gpu -x -q 2>&1 | tail -5
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
