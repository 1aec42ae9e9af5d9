timeout 120 python tools/prof_gather.py --config C1 --rows 1000000 --iters 2 --time 2>&1 | tail -1 | cut -c1-90
timeout 120 python tools/prof_gather.py --config C4 --rows 200000 --iters 2 --time 2>&1 | tail -1 | cut -c1-90
