cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -x -q -k "hash" > gpurun_out/mc_pytest.log 2>&1; echo EXIT=$? >> gpurun_out/mc_pytest.log
for i in 1 2; do
DSRT_HASH_MC=0 python tools/prof_hash.py --mode 3 >> gpurun_out/mc.log 2>&1
python tools/prof_hash.py --mode 3 >> gpurun_out/mc.log 2>&1
done
python tools/prof_hash.py --mode 4 --dtype f16 >> gpurun_out/mc.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:hash_tc_kernel -c 2 --csv --log-file gpurun_out/mc_ncu.csv python tools/prof_hash.py --mode 3 --n 4000000 --reps 1 > gpurun_out/mc_ncu.log 2>&1
DSRT_HASH_MC=0 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:hash_tc_kernel -c 2 --csv --log-file gpurun_out/mc0_ncu.csv python tools/prof_hash.py --mode 3 --n 4000000 --reps 1 > gpurun_out/mc0_ncu.log 2>&1
