cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_envelope.py -m gpu -x -q -k "hash or layout or e2e or end_to_end or cfg0" > gpurun_out/cp_pytest.log 2>&1; echo EXIT=$? >> gpurun_out/cp_pytest.log
python tools/prof_hash.py --mode 3 > gpurun_out/cp.log 2>&1
python tools/prof_hash.py --mode 3 >> gpurun_out/cp.log 2>&1
python tools/prof_hash.py --mode 3 --no-codes >> gpurun_out/cp.log 2>&1
