cd $GRAFT_REPO_ROOT
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; rc=$?; echo "smoke rc=$rc"
tail -3 gpurun_out/smoke.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 600 python -m pytest tests -m gpu -q --timeout 200 --timeout-method=thread -rA > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "PASSED|FAILED|Error|passed|failed" gpurun_out/pytest_gpu.log | tail -30
