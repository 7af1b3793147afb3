export PYTHONPATH=.
L=paper_1810_01967_b200
for v in "" _EMPTY _EMPTY_NOCOPY _EMPTY_NOROT _NOROT; do CBB_TC_CLUSTER=1 CBB_LIB_PATH=$L/libcoverblip_b200$v.so timeout 120 python scripts/probe_mfk.py 2>&1 | tail -1; done
for v in _EMPTY _EMPTY_NOCOPY; do CBB_TC_CLUSTER=2 CBB_LIB_PATH=$L/libcoverblip_b200$v.so timeout 120 python scripts/probe_mfk.py 2>&1 | tail -1 | sed 's/^/csz2 /'; done
