#!/bin/bash
# dev helper: bench the psi tile shape override PLUGIN_PSI_R on the GPU box
for r in 8 4 2; do
  echo "R=$r"; PLUGIN_PSI_R=$r timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['passes'])"
done
