"""Summarise attn_trace output for the v3 kernel (dev tool)."""
import sys
from collections import defaultdict
import statistics as st
ev = defaultdict(dict)
for line in open(sys.argv[1]):
    w, e, it, c = map(int, line.split())
    ev[(w, e)][it] = c
skip = 30
def d(a, b): return (b - a) & 0xffffffff
def ph(w0, e0, w1, e1, shift=0):
    xs = [d(ev[(w0, e0)][i], ev[(w1, e1)][i + shift]) for i in ev[(w0, e0)] if i >= skip and (i + shift) in ev[(w1, e1)]]
    return (round(st.median(xs)), round(st.mean(xs))) if xs else None
for w in (4, 5, 8, 9):
    print(f"softmax warp {w}: S ready->xchg {ph(w,1,w,3)} xchg->P {ph(w,3,w,4)} P->next S ready {ph(w,4,w,1,1)} period {ph(w,1,w,1,1)}")
print("MMA: p_full seen -> S issued (same j+3)", ph(1, 14, 1, 12, 3), " S issued period", ph(1, 12, 1, 12, 1))
print("MMA: S(j) issued -> softmax warp4 sees S(j)", ph(1, 12, 4, 1))
print("softmax warp4 P(j) -> MMA sees p_full(j)", ph(4, 4, 1, 14))
print("MMA p_full(j) -> p_full(j+1)", ph(1, 14, 1, 14, 1))
for w in (4, 8):
    print(f"warp {w}: xchg->exp done {ph(w,3,w,6)} exp->st waited {ph(w,6,w,7)} st->arrived {ph(w,7,w,4)}")
print("MMA pv: p_full seen->V ready", ph(1,14,1,15), "V ready->PV issued", ph(1,15,1,16), "PV issued->K(j+3) ready", ph(1,16,1,17,3), "K ready->S issued", ph(1,17,1,12))
# TMA: load n issued (ev 21, after empty wait); K_{j} is load index j for j<3 else 2j-2; V_j is 2j+3
def kidx(j): return j if j < 3 else 2 * j - 2
xs=[]; ys=[]; zs=[]
for j in range(skip, 400):
    n = kidx(j)
    if n in ev[(0,21)] and j in ev[(1,17)] and n in ev[(0,20)]:
        xs.append(d(ev[(0,21)][n], ev[(1,17)][j]))   # TMA issue -> MMA sees K_j ready
        zs.append(d(ev[(0,20)][n], ev[(0,21)][n]))   # TMA waiting for empty slot
    if (j-3) >= 0 and (j-3) in ev[(1,16)] and n in ev[(0,21)]:
        ys.append(d(ev[(1,16)][j-3], ev[(0,21)][n]) if True else 0)
print("TMA: K_j load issued -> MMA sees K_j ready (median)", st.median(xs) if xs else None,
      " TMA wait for empty slot before K_j", st.median(zs) if zs else None)
