#!/usr/bin/env bash
# Round-2 evidence run on the GPU box (writes gpurun_out/): edge-case tests,
# the default bench line, the bench's launch list (one metric, cold-cache,
# serialised) and `--set full` captures of the hot kernels, each only after
# the plain command exited 0.  Summaries: profiles/summarize.py.
set -u
OUT=${OUT:-gpurun_out}
mkdir -p "$OUT"
timeout 900 python -m pytest tests/test_gpu_edge_cases.py -q -x > "$OUT/r02_edge.log" 2>&1; echo "edge=$?"
timeout 900 python bench.py > "$OUT/r02_bench.json" 2> "$OUT/r02_bench.err"; echo "bench=$?"
P="python bench.py --steps 2 --warmup 1 --no-cpu"
timeout 600 $P > "$OUT/r02_plain.log" 2>&1 || { echo "plain run failed"; exit 1; }
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file "$OUT/r02_launches.csv" $P > "$OUT/r02_ncu_launches.log" 2>&1; echo "launches=$?"
for spec in "pr_tile_k:25:1" "bfs_coop_k:3:1" ${EXTRA_SPECS:-}; do
  k=${spec%%:*}; rest=${spec#*:}; s=${rest%%:*}; c=${rest#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$k" -s "$s" -c "$c" \
    -o "$OUT/r02_full_$k" $P > "$OUT/r02_ncu_$k.log" 2>&1
  echo "$k=$?"
done
