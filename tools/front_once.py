"""Two front-door calls (config 2 seeds 1, 2): profiling target for the launch list."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_08963_b200 as mdg  # noqa: E402

dev = mdg.Device(0)
for s in (1, 2):
    r = mdg.min_weight(mdg.gen_matrix(128, 64, s, True), 128, 10, 1, device=dev)
    print(s, r.d, r.launches, flush=True)
