cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_search.py tests/test_envelope.py -m gpu -x -q > gpurun_out/cl_pytest.log 2>&1; echo EXIT=$? >> gpurun_out/cl_pytest.log
for i in 1 2; do
DSRT_ALL_CLUSTER=0 python tools/prof_score.py --sets 1000000 --qsets 1024 --L 32 --C 8 --reps 3 >> gpurun_out/cl.log 2>&1
python tools/prof_score.py --sets 1000000 --qsets 1024 --L 32 --C 8 --reps 3 >> gpurun_out/cl.log 2>&1
done
python tools/prof_score.py --sets 100000 --qsets 1000 --L 64 --C 7 --reps 3 >> gpurun_out/cl.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --clock-control none -k regex:score_all_kernel -c 1 --csv --log-file gpurun_out/cl_ncu.csv python tools/prof_score.py --sets 1000000 --qsets 1024 --L 32 --C 8 --reps 1 > gpurun_out/cl_ncu.log 2>&1
DSRT_ALL_CLUSTER=0 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --clock-control none -k regex:score_all_kernel -c 1 --csv --log-file gpurun_out/cl0_ncu.csv python tools/prof_score.py --sets 1000000 --qsets 1024 --L 32 --C 8 --reps 1 > gpurun_out/cl0_ncu.log 2>&1
