timeout 300 python tools/probes/e2e_probe.py 2>&1 | grep -v "flush none"
