cd $GRAFT_REPO_ROOT
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "small or golden or agg or prefilter or tinytable or layout or hash_golden or cfg0" > gpurun_out/san1.log 2>&1; echo EXIT=$? >> gpurun_out/san1.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_envelope.py tests/test_gpu_search.py -m gpu -x -q -k "not concurrent" > gpurun_out/san2.log 2>&1; echo EXIT=$? >> gpurun_out/san2.log
