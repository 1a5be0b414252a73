cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests/test_pd_gpu.py -x -q --durations=5 > gpurun_out/pytest_pd.log 2>&1; tail -25 gpurun_out/pytest_pd.log
