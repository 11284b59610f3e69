"""Summarise tools/ubench/attn_trace output: per-iteration phase durations of
the softmax warps and the MMA issuer of one attention CTA (dev tool)."""
import sys
from collections import defaultdict
import statistics as st

ev = defaultdict(dict)  # (warp, ev) -> {it: clk}
for line in open(sys.argv[1]):
    w, e, it, c = map(int, line.split())
    ev[(w, e)][it] = c
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 20


def d(a, b):
    return (b - a) & 0xffffffff


def phase(w, e0, e1, shift=0):
    xs = [d(ev[(w, e0)][i], ev[(w, e1)][i + shift]) for i in ev[(w, e0)]
          if i >= skip and (i + shift) in ev[(w, e1)]]
    return (round(st.median(xs)), round(st.mean(xs))) if xs else None


for w in (4, 5, 8, 9):
    print(f"softmax warp {w}: wake->ld {phase(w,1,2)} ld->max {phase(w,2,3)} max->P0 {phase(w,3,4)} "
          f"P0->P1 {phase(w,4,5)} P1->next wake {phase(w,5,1,1)} period {phase(w,1,1,1)}")
# MMA: per tile t, p_full(t,half0) wait done -> S(t) issued, S issued -> next p_full
for t in (0, 1):
    print(f"mma tile {t}: pfull0->pfull1 {phase(1,14+2*t,15+2*t)} pfull1->sfree {phase(1,15+2*t,10+t,1)} "
          f"sfree->S issued {phase(1,10+t,12+t)} period {phase(1,12+t,12+t,1)}")
# cross: softmax0 P1 ready (warp 4 ev 5 it i) vs MMA observed p_full(0, half1) (ev 15, n_pv)
print("S0 issued -> softmax0 wake:", phase(1, 12, 1) if False else None)
xs = []
for i in ev[(4, 1)]:
    if i >= skip and i in ev[(1, 12)]:
        xs.append(d(ev[(1, 12)][i], ev[(4, 1)][i]))
print("S(t0) commit issued -> warp4 wakes (S done):", round(st.median(xs)) if xs else None)
xs = []
for i in ev[(4, 5)]:
    if i >= skip and (i) in ev[(1, 15)]:
        xs.append(d(ev[(4, 5)][i], ev[(1, 15)][i]))
print("warp4 P1 arrive -> MMA sees p_full(0,1):", round(st.median(xs)) if xs else None)
for w in (4, 8):
    print(f"warp {w}: max->exp0 done {phase(w,3,6)} exp0 done->st0 waited {phase(w,6,8)} st0->arrive0 {phase(w,8,4)} "
          f"arrive0->exp1 done {phase(w,4,7)} exp1 done->st1 waited {phase(w,7,9)}")
