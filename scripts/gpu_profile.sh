cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
# launch list (cold, serialised) of 2 forward+backward frames after 2 warm-up frames
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_frame.py --frames 4 --backward > gpurun_out/launches.log 2>&1; echo "launch list rc=$?"
# full sets of the top kernels (one launch each, after warm-up)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_forward|k_backward|k_preprocess|k_tiles_scatter" -s 8 -c 4 -o gpurun_out/prof_frame python scripts/profile_frame.py --frames 4 --backward > gpurun_out/prof.log 2>&1; echo "full rc=$?"
timeout 600 ncu --set full --clock-control none -k regex:"Onesweep" -s 4 -c 4 -o gpurun_out/prof_sort python scripts/profile_frame.py --frames 3 > gpurun_out/prof_sort.log 2>&1; echo "sort rc=$?"
ls -la gpurun_out
