#!/bin/bash
# Block-parallel exoneration sweep (CSG_EXO_BLOCK_SWEEP=1): GPU suite + C3
# paths + timing against the warp sweep.
set -u
O=gpurun_out/${1:-exo}
mkdir -p "$O"
export CSG_EXO_BLOCK_SWEEP=1
timeout 1200 python -m pytest tests -m gpu -x -q > "$O/pytest_gpu.log" 2>&1
echo "pytest_gpu(block) $?" >> "$O/status"
timeout 500 python scripts/c3_paths.py > "$O/c3_paths.json" 2> "$O/c3_paths.err"
echo "c3_paths(block vs warp+slow) $? $(tail -1 $O/c3_paths.json)" >> "$O/status"
for V in 1 0; do
  if [ $V = 1 ]; then export CSG_EXO_BLOCK_SWEEP=1; else unset CSG_EXO_BLOCK_SWEEP; fi
  TAG=blk$V timeout 300 python scripts/kbench.py > "$O/kbench_blk$V.txt" 2>&1
  echo "kbench block=$V $(grep k_exonerate $O/kbench_blk$V.txt)" >> "$O/status"
  timeout 400 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu --no-jsonl > "$O/bench_c3_blk$V.json" 2> "$O/bench_c3_blk$V.err"
  echo "c3 block=$V $(python scripts/roofline_line.py $O/bench_c3_blk$V.json 2>&1 | tail -1) $(python -c "import json;d=json.load(open('$O/bench_c3_blk$V.json'));s=d['roofline']['share_of_step'];print('exo ms', round(s.get('k_exonerate',0)*d['ms_per_step'],2))" 2>&1)" >> "$O/status"
done
cat "$O/status"
