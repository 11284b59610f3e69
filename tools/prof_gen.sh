# ncu launch times of a short c4 generation (dev tool): every kernel after the
# prompt prefill (decode attention, merge, GEMMs + split-K reduce, norms, RoPE,
# sampling) for 2 decode steps.
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k "regex:dec_|sample_|decode_embed|splitk|gemm|rmsnorm|rope" -c 2000 --csv python tools/gen_once.py 2>/dev/null > gpurun_out/gen_launches.csv
wc -l gpurun_out/gen_launches.csv
