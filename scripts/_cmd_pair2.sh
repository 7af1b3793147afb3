export PYTHONPATH=.
L=paper_1810_01967_b200
for v in _EMPTY _EMPTY_NOCOPY; do for p in 0 1; do CBB_TC_PAIR=$p CBB_LIB_PATH=$L/libcoverblip_b200$v.so timeout 100 python scripts/probe_mfk.py 2>&1 | tail -1 | sed "s/^/pair=$p /"; done; done
echo "== trace pair"; timeout 120 python scripts/trace_tc.py 2>&1 | tail -22
