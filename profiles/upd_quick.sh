#!/bin/bash
# batch-update timings at the four config-5 sizes (3 reps each; rep 0 warms)
for s in 10000 100000 1000000 10000000; do python profiles/run_updates.py --size $s --reps 3 2>&1 | tail -2; done
