#!/bin/bash
# 3-d colour-path Jacobian: 1 / 2 / 4 tangents per flux pass (three builds)
mkdir -p gpurun_out
for lib in "" scratch/libpint_nt2.so scratch/libpint_nt4.so; do
  if [ -n "$lib" ]; then export PINT_LIB=$PWD/$lib; else unset PINT_LIB; fi
  timeout 600 python tools/elem_ab.py --cases c4 --variants "" | sed "s|^|{\"lib\": \"$lib\"} |" >> gpurun_out/az_elem.jsonl 2>> gpurun_out/az_elem.err
  timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline 2>> gpurun_out/az.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'lib': '$lib', 'value': d['value'], 'solver': d['solver'], 'parity': d['parity'] and d['parity']['pass']}))" >> gpurun_out/az_ab.jsonl
done
true
