cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/full_pytest.log 2>&1; echo EXIT=$? >> gpurun_out/full_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo EXIT=$? >> gpurun_out/smoke.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo EXIT=$? >> gpurun_out/bench_final.err
timeout 600 python bench.py --config 2 --steps 20 --warmup 5 > gpurun_out/b2.json 2> gpurun_out/b2.err
