set -x
O=gpurun_out/r02e; mkdir -p $O
md5sum paper_2510_08055_b200/_lib/liblpmoe.so > $O/md5.txt
timeout 900 python -m pytest tests/test_gpu_moe.py -x -q -k "decode or qwen_layer or tiny_config or launch_count or batch_invariance or graph or experimental" > $O/pytest_decode.log 2>&1
for T in 1 2 4 8 16; do timeout 120 python bench.py --tokens $T --steps 30 --no-cpu-baseline; done > $O/bench_decode.jsonl 2> $O/bench_decode.err
for T in 1 8; do LP_T=$T LP_TINY_ITEMS=1 timeout 120 python tools/trace_layer.py > $O/trace_T$T.txt 2>&1; done
