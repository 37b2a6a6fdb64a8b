#!/bin/bash
# K1 hi/lo hash: parity tests, then timing of the library and of timing-only variants
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -k "hash or tc or cfg2" > $O/exp_hash_tests.log 2>&1; echo EXIT=$? >> $O/exp_hash_tests.log
: > $O/exp_hash.txt
for v in base $VARIANTS; do
  if [ $v = base ]; then L=""; else L="paper_2210_15748_b200/csrc/variant_$v.so"; fi
  for dt in bf16 fp16; do
    M=3; [ $dt = fp16 ] && M=4
    DSRT_LIB=$L python tools/prof_hash.py --mode $M --dtype $dt --reps 20 >> $O/exp_hash.txt 2>&1
    DSRT_LIB=$L python tools/prof_hash.py --mode $M --dtype $dt --reps 20 --no-codes >> $O/exp_hash.txt 2>&1
  done
done
