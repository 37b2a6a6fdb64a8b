#!/bin/bash
# Round check on one B200: -m gpu tests, smoke, the driver's two bench arms with wall-clock times.
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out
S=$(date +%s)
timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo PYTEST_EXIT=$? >> $O/pytest_gpu.log
echo "pytest_s=$(( $(date +%s) - S ))" > $O/validate_times.txt
S=$(date +%s)
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > $O/smoke.log 2>&1; echo SMOKE_EXIT=$? >> $O/smoke.log
echo "smoke_s=$(( $(date +%s) - S ))" >> $O/validate_times.txt
S=$(date +%s)
timeout 1200 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/bench_ref.json 2> $O/bench_ref.err
echo "ref_s=$(( $(date +%s) - S ))" >> $O/validate_times.txt
S=$(date +%s)
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_default.json 2> $O/bench_default.err
echo "bench_s=$(( $(date +%s) - S ))" >> $O/validate_times.txt
