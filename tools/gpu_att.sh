# measured-attention serving on one B200: attention micro-benchmark, executor tests, then C3 with
# pooled KV + whole-iteration decode graphs
set -x
mkdir -p gpurun_out
python tools/attn_micro.py > gpurun_out/attn_micro.txt 2>&1
python -m pytest tests/test_gpu_executor.py -q -x 2>&1 | tail -5
