"""TEST INFRASTRUCTURE: regenerate tests/golden/ fixtures.

* rng_golden.json — printed by oracle/_ref/ref_rng_golden, a tool compiled
  from the REFERENCE's own proj/include/cprand/rng.hpp (oracle/Makefile
  target `ref`). It pins seeded_engine + the libstdc++ distributions the
  reference consumes; tests/test_oracle_golden.py checks the oracle against it.
* known_answers.json — inline constants from the reference's test suite,
  each with the file:line it comes from.

Run here (needs /root/reference):  python oracle/make_golden.py
"""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
GOLD = os.path.join(ROOT, "tests", "golden")


def main() -> int:
    if not os.path.isdir("/root/reference"):
        print("make_golden: /root/reference absent; nothing to regenerate")
        return 0
    subprocess.check_call(["make", "-s", "-C", HERE, "ref"])
    out = subprocess.check_output([os.path.join(HERE, "_ref", "ref_rng_golden")], text=True)
    doc = json.loads(out)
    os.makedirs(GOLD, exist_ok=True)
    with open(os.path.join(GOLD, "rng_golden.json"), "w") as f:
        json.dump(doc, f, indent=0)
    known = {
        "unfold_column_index": {
            "src": "proj/tests/test_tensor.cpp:68-73",
            "dims": [3, 4, 5], "idx": [1, 2, 3], "mode": 0, "want": 14},
        "default_sample_count": {
            "src": "proj/tests/test_sampling.cpp:25-31",
            "cases": [[1, 10], [2, 14], [5, 80], [6, 108]]},
        "layout_strides": {
            "src": "proj/tests/test_tensor.cpp:40-56",
            "dims": [3, 4, 5], "strides": [1, 3, 12], "entry": [[2, 3, 4], 47]},
        "should_stop_sequence": {
            "src": "proj/tests/test_sampling.cpp:202-232",
            "stall_limit": 3, "max_iters": 100,
            "fits": [0.5, 0.4, 0.45, 0.4], "stop": [0, 0, 0, 1], "reason_last": 3},
        "readme_run": {
            "src": "proj/README.md:58-65",
            "dims": [50, 50, 50], "rank": 5, "collinearity": 0.5, "noise": 0.01,
            "seed": 3, "samples": 80, "iters": 53, "fit_prefix": "0.98870",
            "stop": "best_fit_stall",
            "note": "generator is the reference gen_problem (Eigen HouseholderQR): "
                    "restated, so only tolerance-level agreement is expected"},
    }
    with open(os.path.join(GOLD, "known_answers.json"), "w") as f:
        json.dump(known, f, indent=1)
    print("wrote", os.listdir(GOLD))
    return 0


if __name__ == "__main__":
    sys.exit(main())
