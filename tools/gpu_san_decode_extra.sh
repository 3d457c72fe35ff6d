bash tools/gpu_san_decode.sh
O=gpurun_out/san2
for rep in 1 2; do for T in 2048 8224; do timeout 300 python bench.py --tokens $T --steps 30 --no-cpu-baseline; done; done > $O/bench_large.jsonl 2>$O/bench_large.err
