#!/bin/bash
# Final-tree check on one B200: full GPU suite, smoke, config-2 bench line, decode-size lines.
O=gpurun_out/final; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench.jsonl 2>$O/bench.err
for T in 1 8; do timeout 300 python bench.py --tokens $T --steps 30 --no-cpu-baseline; done > $O/bench_decode.jsonl 2>$O/bench_decode.err
