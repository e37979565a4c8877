for s in 10000 100000 1000000 10000000; do python profiles/run_updates.py --size $s --reps 3 2>&1 | tail -1; done
