cd $GRAFT_REPO_ROOT
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_frame.py --frames 3 --backward > /dev/null 2>&1; echo "ncu rc=$?"
