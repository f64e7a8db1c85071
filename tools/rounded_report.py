"""plugin_h on the rounded BASELINE configs (inputs.ROUNDED) and cfg4 against their goldens:
relative errors per field, one JSON line each (dev helper; PLUGIN_LIB_PATH selects A/B variants)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1505_02100_b200 import inputs  # noqa: E402
from paper_1505_02100_b200 import plugin as P  # noqa: E402

KEYS = ("psi6_z", "psi4_z", "h", "g2")
for name in list(inputs.ROUNDED) + ["4"]:
    g = json.load(open(os.path.join(ROOT, "tests", "golden", f"cfg{name}.json")))
    x = inputs.rounded_data(name) if name in inputs.ROUNDED else inputs.config_data(int(name))
    r = P.plugin_h_sync(torch.from_numpy(x).cuda())
    print(json.dumps({"config": name, "lib": os.path.basename(P.LIB_PATH),
                      "rel_err": {k: (r[k] - g[k]) / abs(g[k]) for k in KEYS}}), flush=True)
