"""Extended randomised parity sweep (same generator as tests/test_gpu_fuzz.py, more seeds).

    python scripts/fuzz_many.py N_SMALL N_LARGE
"""
import os
import sys
import traceback

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.test_gpu_fuzz import test_random_case_vs_oracle  # noqa: E402

n_small, n_large = int(sys.argv[1]), int(sys.argv[2])
fails = []
cases = [(s, False) for s in range(1000, 1000 + n_small)] + [(s, True) for s in range(1000, 1000 + n_large)]
for seed, large in cases:
    try:
        test_random_case_vs_oracle(seed, large)
    except Exception as exc:  # noqa: BLE001
        fails.append((seed, large, repr(exc)[:300]))
        traceback.print_exc(limit=2)
print(f"{len(cases)} cases, {len(fails)} failures")
for f in fails:
    print("FAIL", f)
