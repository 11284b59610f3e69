# attention: determinism, parity tests, CUDA-event throughput per exp2 share
set -x
timeout 300 python tools/attn_det.py
timeout 600 python -m pytest tests/test_attention_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 900 python tools/attn_perf.py 0 8
