#!/bin/bash
# psi pass time per n for each rows-per-thread R of the work-unit kernel (PLUGIN_PSI_R), and
# the default choice; output gpurun_out/$1_sweep.jsonl
out=gpurun_out/${1:-units}_sweep.jsonl
: > $out
NS="4096 8192 12000 16384 24576 32768 49152 65536 98304 131072 196608 262144 524288"
python tools/psi_time.py $NS >> $out
for R in 1 2 4 8; do PLUGIN_PSI_R=$R python tools/psi_time.py $NS >> $out; done
