cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/q_pytest.log 2>&1; tail -2 gpurun_out/q_pytest.log
