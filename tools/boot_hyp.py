"""Time the Set_hyp bootstrap alone (bench.bench_bootstrap_set_hyp) and print its JSON."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2302_02407_b200 as hy  # noqa: E402
import synth  # noqa: E402

ctx = hy.Context(**synth.PARAMS["hyp"], device=0, max_batch=int(os.environ.get("HY_BENCH_BATCH", "64")))
print(json.dumps(bench.bench_bootstrap_set_hyp(ctx, int(sys.argv[1]) if len(sys.argv) > 1 else 3), indent=1))
torch.cuda.synchronize()
