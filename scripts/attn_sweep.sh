#!/bin/bash
# time the attention kernel for several library builds (BLADE_LIB variants)
for lib in "$@"; do
  r=$(BLADE_LIB=$lib timeout 200 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4f ms attn  %.4f ms mask  frac %.3f  clk %s' % (d['ms_attn'], d['ms_mask'], d['roofline']['frac'], d['clocks']['sm_mhz']))")
  echo "$lib: $r"
done
