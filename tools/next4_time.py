"""Dev tool: NEXT-3 / NEXT-4 block timings (bench.py's resblock_levels / temporal_levels) on the
configs[2] request, without the rest of the bench.  Prints one JSON object."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_18672_b200 as sp  # noqa: E402
from paper_2511_18672_b200.step import RefinementStep  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
sp.load()
st = RefinementStep(bench.step_config(bench.WORKLOADS["configs2"]["means"]), bench.make_batch("configs2"), dev, sp)
st.run()
torch.cuda.synchronize()
out = {"temporal": bench.temporal_levels(torch, st)}
if "--resblock" in sys.argv:
    out["resblock"] = bench.resblock_levels(torch, st)
print(json.dumps(out))
