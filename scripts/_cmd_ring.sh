export PYTHONPATH=.
for v in f16noscreen f16nold; do echo "== $v"; CBB_LIB_PATH=scratch_libs/$v.so timeout 300 python scripts/probe_split_mode.py cfg1 2>&1 | grep -v "^$" | grep "tcgen05 "; done
