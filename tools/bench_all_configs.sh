#!/bin/bash
# Every config line (with its cpu_baseline) + the reference arm; outputs in gpurun_out/.
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out
timeout 900 python bench.py --config 3 --steps 20 --warmup 5 > $O/b_cfg3.json 2> $O/b_cfg3.err
timeout 600 python bench.py --config 2 --steps 20 --warmup 5 > $O/b_cfg2.json 2> $O/b_cfg2.err
timeout 600 python bench.py --config 1 --steps 20 --warmup 5 > $O/b_cfg1.json 2> $O/b_cfg1.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $O/b_ref.json 2> $O/b_ref.err
