# A/B: CTA-specialised hybrid exp for the r = 4, R = 8 pass (the last 1/k of the CTAs evaluate every
# exp on the FMA pipe, -DPSI_CTA_HYB=k), cfg4 pass times and parity.  Not kept: psi4 123 -> 160 ms (k = 2)
# and 140 ms (k = 4); profiles/r04l_ab_cta_hybrid_exp*.jsonl
set -u
for rep in 1 2; do
  for lib in libplugin.so libplugin_ctahyb2.so libplugin_ctahyb4.so; do
    PLUGIN_LIB_PATH=$PWD/paper_1505_02100_b200/$lib python tools/psi_graph_time.py 1048576 | sed "s/^{/{\"variant\": \"$lib\", /" >> gpurun_out/ab_ctahyb.jsonl
  done
done
for lib in libplugin_ctahyb2.so libplugin_ctahyb4.so; do
  PLUGIN_LIB_PATH=$PWD/paper_1505_02100_b200/$lib timeout 300 python tools/parity_report.py | sed "s/^{/{\"variant\": \"$lib\", /" >> gpurun_out/ab_ctahyb_parity.jsonl
done
