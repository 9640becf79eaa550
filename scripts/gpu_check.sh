cd $GRAFT_REPO_ROOT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -3 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -rA > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "PASSED|FAILED|Error|passed|failed" gpurun_out/pytest_gpu.log | tail -30
