#!/bin/bash
# dev helper: bench each tools/variants/*.so (PLUGIN_LIB_PATH override)
for f in tools/variants/*.so; do
  echo -n "$f "; PLUGIN_LIB_PATH=$PWD/$f timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); p=d['passes']; print(round(d['value'],1), round(d['roofline']['frac'],4), round(p['psi6_gpairs_s'],1), round(p['psi4_gpairs_s'],1))"
done
