#!/bin/bash
# quick N=1 bench summary: value, e2e, per-kernel-class profile
timeout 300 python bench.py --no-cpu-baseline "$@" 2>gpurun_out/qb.err | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print(d['value'], d['e2e']['value'] if d.get('e2e') else None, d['ms_per_step'], d.get('clocks'))
print({k:(v['launches'], round(v['ms'],2), round(v['rate'])) for k,v in d['roofline']['kernels'].items()})"
