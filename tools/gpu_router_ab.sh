set -x
O=gpurun_out/rt; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_moe.py -x -q -k "size_sweep" > $O/pytest_sweep.log 2>&1
for cs in 0 2; do for T in 2048 8224; do LPMOE_ROUTER_CS=$cs timeout 200 python bench.py --tokens $T --steps 20 --no-cpu-baseline; done; done > $O/bench_router.jsonl 2>$O/bench_router.err
