#!/bin/bash
# Device JSONL ingest on one GPU: its parity tests, a bench line (with the
# e2e.jsonl file measurement), and one ncu capture of the parse kernel.
#   gpurun --timeout 1800 -- bash scripts/gpu_jsonl.sh <tag>
set -u
O=gpurun_out/${1:-jsonl}
mkdir -p "$O"
timeout 900 python -m pytest tests/test_jsonl_device.py tests/test_abi.py -x -q > "$O/pytest_jsonl.log" 2>&1
echo "pytest jsonl $?" >> "$O/status"
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > "$O/bench.json" 2> "$O/bench.err"
echo "bench $?" >> "$O/status"
cat > /tmp/jl.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
from paper_2509_03018_b200 import engine as E
import glob
p = sorted(glob.glob("/tmp/collsight_c2_*.jsonl"))[0]
s = E.TraceStore()
for _ in range(3):
    s.clear(); assert s.append_jsonl_file(p)
print(len(s))
PY
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_jsonl" -s 3 -c 3 \
    -o "$O/prof_jsonl" python /tmp/jl.py > "$O/ncu.log" 2>&1
echo "ncu $?" >> "$O/status"
cat "$O/status"
