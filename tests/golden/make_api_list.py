"""Record the reference package's public names (attnreuse.__all__) as a fixture.

Run in the build container, where the reference is importable:
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_api_list.py
The CPU test test_host_cpu.py::test_public_names_cover_reference diffs the package's
__all__ against it (minus the out-of-scope names listed in the fixture).
"""

import json
import os

import attnreuse

OUT_OF_SCOPE = {
    # offline LPT scheduling simulator (sched.py), SURVEY.md §2.1 OUT OF SCOPE
    "Plan": "sched.py", "WorkItem": "sched.py", "baselines": "sched.py", "gen_skewed_spans": "sched.py",
    "naive_makespan": "sched.py", "optimal_makespan": "sched.py", "perfect_makespan": "sched.py",
    "plan_lpt": "sched.py",
    # tau calibration utility (matching.py:178-199, scipy), SURVEY.md §2.1 OUT OF SCOPE
    "calibrate_tau": "matching.py:178-199", "chi2_cdf": "matching.py:178-199",
}

if __name__ == "__main__":
    out = {"reference_all": sorted(attnreuse.__all__), "out_of_scope": OUT_OF_SCOPE}
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_api.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print(path, len(out["reference_all"]))
