set -x
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider --durations=15 > gpurun_out/r2a_pytest.log 2>&1
tail -30 gpurun_out/r2a_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1
tail -3 gpurun_out/r2a_smoke.log
