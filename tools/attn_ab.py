"""A/B of attention-forward variants selected by environment variables
(dev tool): python tools/attn_ab.py VAR val1 val2 ... — each shape runs the
variants interleaved, MRSP_PERF_REPS times (clocks drift under the power cap)."""
import json
import math
import os
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from tools.attn_perf import bench  # noqa: E402

if __name__ == "__main__":
    var, vals = sys.argv[1], sys.argv[2:]
    reps = int(os.environ.get("MRSP_PERF_REPS", "3"))
    shapes = [(32768, 28, 4), (16421 + 8 * 1024, 28, 4, 16421, 1024),
              (131109 + 8 * 1011, 28, 4, 131109, 1011)]
    for args in shapes:
        for rep in range(reps):
            for v in vals:
                os.environ[var] = v
                r = bench(*args, iters=2 if args[0] > 100000 else 5)
                r[var], r["rep"] = v, rep
                print(json.dumps(r), flush=True)
