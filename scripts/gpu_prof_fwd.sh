cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_forward|k_backward" -s 2 -c 2 -o gpurun_out/prof_fwd python scripts/profile_frame.py --frames 3 --backward > gpurun_out/prof_fwd.log 2>&1; echo "full rc=$?"
