# ncu launch times of a short c4 generation in graph mode (dev tool): every
# kernel node of the last decode-step graph replay, warm caches
# (--cache-control none), clocks as the driver left them.
python - > /tmp/gen4.py <<'PY'
print('''import sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2507_07966_b200 import engine as E
w = E.workloads()["c4"]; c = w.cfg
eng = E.Engine(c, sp=1, with_ref=False)
pix = torch.from_numpy(E.gen_video(1, w.frames, 3 * c.image_size ** 2)).cuda()
eng.encode("v", pix)
eng.generate("v", np.arange(10, 47, dtype=np.int32), 8, 4, seed=1)
torch.cuda.synchronize()''')
PY
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --cache-control none --clock-control none \
  -k "regex:dec_|sample_|decode_|splitk|gemm|rmsnorm|rope" -c 3000 --csv python /tmp/gen4.py 2>/dev/null > gpurun_out/gen_graph_launches.csv
wc -l gpurun_out/gen_graph_launches.csv
