#!/bin/bash
# ncu --set full of every library kernel that matters in one C2 fwd+bwd frame (frame 2, after warm-up).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-prof}
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"${KREGEX:-k_forward|k_backward|k_finalize|k_preprocess|k_rows_scatter|k_tiles_scatter|k_fixup}" -s ${SKIP:-6} -c ${COUNT:-6} \
  -o gpurun_out/$TAG python scripts/profile_frame.py --frames 3 --backward > gpurun_out/$TAG.log 2>&1; echo "ncu full rc=$?"
tail -3 gpurun_out/$TAG.log
