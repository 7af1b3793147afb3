export PYTHONPATH=.
timeout 600 python scripts/probe_split_mode.py small cfg1 coh coh20 2>&1 | grep -v Warning
