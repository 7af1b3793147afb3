export PYTHONPATH=.
L=paper_1810_01967_b200
for v in "" _EMPTY; do CBB_LIB_PATH=$L/libcoverblip_b200$v.so timeout 100 python scripts/probe_mfk.py 2>&1 | tail -1; done
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
