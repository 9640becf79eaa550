cd $GRAFT_REPO_ROOT
for defs in "$@"; do
  GEER_NVCC_DEFS="$defs" python -m paper_2505_24053_b200.build --force > /dev/null 2>&1 || { echo "build failed: $defs"; continue; }
  echo "== $defs: $(timeout 120 python scripts/stage_times.py 2>/dev/null | tail -1)"
done
