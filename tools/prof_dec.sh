# ncu of the tcgen05 decode-attention launches of a c4 generation (dev tool)
cat > /tmp/gen_once.py <<'PY'
import sys
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
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio \
  --clock-control none -k "regex:dec_attn_tc|dec_merge|gemm" --launch-skip 114 -c 12 --csv python /tmp/gen_once.py 2>/dev/null | grep -E "dec_attn_tc|dec_merge|gemm" > gpurun_out/dec_ncu.csv
wc -l gpurun_out/dec_ncu.csv
