"""Dump the reference's Butcher tableaux (tableaux.py:114-155) as exact
float hex strings into tableaux.json.  Build container only (imports
/root/reference/pkg/src); the JSON travels.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_tableaux.py
"""
import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

import numpy as np  # noqa: E402
from irkmg.tableaux import registry_keys, tableau_lookup  # noqa: E402

out = {}
for fam, s in registry_keys():
    t = tableau_lookup(fam, s)
    out[f"{fam}:{s}"] = {k: [float(v).hex() for v in np.asarray(getattr(t, k), float).ravel()]
                         for k in ("A", "b", "c")}
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "tableaux.json"), "w") as fh:
    json.dump(out, fh, indent=1, sort_keys=True)
print(sorted(out))
