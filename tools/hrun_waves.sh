cd $GRAFT_REPO_ROOT
for w in 8 16 32 4; do
  DSRT_ALL_WAVES=$w timeout 600 python bench.py --sets 2000000 --steps 3 --warmup 3 --no-cpu-baseline --no-extra --e2e-steps 1 > gpurun_out/w$w.json 2> gpurun_out/w$w.err
  DSRT_ALL_WAVES=$w DSRT_PROFILE_STEPS=1 ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:score_all_kernel --csv --log-file gpurun_out/w${w}_ncu.csv python bench.py --sets 2000000 --steps 1 --warmup 3 --no-cpu-baseline --no-extra --e2e-steps 1 > gpurun_out/w${w}_ncu.log 2>&1
done
