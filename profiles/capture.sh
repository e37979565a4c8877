#!/usr/bin/env bash
# Profiling recipe (run on the GPU box under gpurun; writes gpurun_out/).
# 1. the plain command must exit 0 first (B200_PROFILING.md rule),
# 2. launch list of the whole bench (one metric, cold-cache, serialised),
# 3. one `--set full` capture per hot kernel, skipping warm-up launches.
# Summaries for the repo: python profiles/summarize.py full|launches ...
set -u
OUT=${OUT:-gpurun_out}
TAG=${TAG:-r01}
mkdir -p "$OUT"
P="python bench.py --steps 2 --warmup 1 --no-cpu"
timeout 600 $P > "$OUT/${TAG}_plain.log" 2>&1 || { echo "plain run failed"; exit 1; }
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file "$OUT/${TAG}_launches.csv" $P > "$OUT/${TAG}_ncu_launches.log" 2>&1
echo "launches=$?"
# kernel regex : launches to skip (past warm-up / first graph) : count
for spec in "pr_iter_k:25:1" "pull_k:2:2" "push_k:3:2" "expand_k:6:3" "apply_flags_k:2:1" \
            "tc_count_k:0:1" "cc_sample_k:0:1" "DeviceRadixSortOnesweepKernel:12:1" "rmat_keys_k:0:1" \
            ${EXTRA_SPECS:-}; do
  k=${spec%%:*}; rest=${spec#*:}; s=${rest%%:*}; c=${rest#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$k" -s "$s" -c "$c" \
    -o "$OUT/${TAG}_full_$k" $P > "$OUT/${TAG}_ncu_$k.log" 2>&1
  echo "$k=$?"
done
