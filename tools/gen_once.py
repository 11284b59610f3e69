"""One short c4 generation (prompt prefill + 2 decode steps) — target for ncu captures."""
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2507_07966_b200 import engine as E

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
w = E.workloads()[name]
c = w.cfg
eng = E.Engine(c, sp=1, with_ref=False)
pix = torch.from_numpy(E.gen_video(1, w.frames, 3 * c.image_size ** 2)).cuda()
eng.encode("v", pix)
eng.generate("v", np.arange(10, 10 + w.n_question, dtype=np.int32), 8, 2, seed=1)
torch.cuda.synchronize()
