#!/bin/bash
# decode kernel A/B over one env knob: tools/gpu_decode_ab.sh TAG KNOB "V1 V2 ..." "T1 T2 ..." (interleaved x2)
O=gpurun_out/$1; KNOB=$2; mkdir -p $O
for rep in 1 2; do for v in $3; do for T in $4; do
  env $KNOB=$v timeout 120 python bench.py --tokens $T --steps 40 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$KNOB=$v', 'T=%d' % d['config']['tokens'], round(d['value'],1), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done; done; done > $O/ab.txt 2> $O/ab.err
cat $O/ab.txt
