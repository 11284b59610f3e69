# ncu launch times of one c4 decode step (dev tool): decode-only kernels, and
# the GEMMs of the first step (after the 112 GEMMs of the prompt prefill)
cat > /tmp/gen_once.py <<'PY'
import sys, pathlib
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2507_07966_b200 import engine as E
w = E.workloads()["c4"]; c = w.cfg
eng = E.Engine(c, sp=1, with_ref=False)
pix = torch.from_numpy(E.gen_video(1, w.frames, 3 * c.image_size ** 2)).cuda()
eng.encode("v", pix)
eng.generate("v", np.arange(10, 47, dtype=np.int32), 8, 2, seed=1)
torch.cuda.synchronize()
PY
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:dec_|sample_|decode_embed|rmsnorm|rope" -c 400 --csv python /tmp/gen_once.py 2>/dev/null | grep -E "dec_|sample_|decode_embed|rmsnorm|rope" > gpurun_out/gen_dec.csv
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:gemm" --launch-skip 114 -c 113 --csv python /tmp/gen_once.py 2>/dev/null | grep gemm > gpurun_out/gen_gemm.csv
wc -l gpurun_out/gen_dec.csv gpurun_out/gen_gemm.csv
