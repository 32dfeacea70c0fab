#!/bin/bash
for f in gpurun_out/trace_$1_*c?.json gpurun_out/trace_$1_c?.json; do [ -f $f ] && python -c "
import json,sys; d=json.load(open('$f')); print('$f'.split('/')[-1], 'ms/iter %.4f'%d['ms_per_iter'], 'assign %.3f other %.3f'%(d['timing']['assign_ms'], d['timing']['other_ms']))"; done 2>/dev/null | sort -u
