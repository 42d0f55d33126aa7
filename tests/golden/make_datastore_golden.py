"""Golden vectors for the datastore (run here, where the reference exists):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_datastore_golden.py
Writes tests/golden/datastore.json + tests/golden/ds_fixture/ (a 4-sample
mse and a 2-sample xent HSB1 fixture written by the reference itself) so the
datastore tests never need /root/reference at run time."""
import json
import os
import shutil
from pathlib import Path

import numpy as np

from voxpar import datastore as R
from voxpar.tensor import ProcessGrid

here = Path(__file__).resolve().parent
out = {}
out["perm"] = {f"{s},{e},{t}": list(R.epoch_schedule(s, e, t, 2, 1).perm)
               for s, e, t in ((0, 0, 10), (0, 1, 10), (3, 2, 17), (1, 0, 4))}
sched = R.epoch_schedule(0, 0, 8, 4, 2)
man_dir = here / "ds_fixture" / "mse"
if man_dir.exists():
    shutil.rmtree(man_dir)
man = R.generate_fixture(str(man_dir), 8, (2, 4, 6, 8), loss="mse", seed=5)
out["owner_map_8_4_2"] = {str(k): v for k, v in R.build_owner_map(man, ProcessGrid(2, 1, 1, 1), sched).items()}
out["targets"] = man.targets().tolist()
xdir = here / "ds_fixture" / "xent"
if xdir.exists():
    shutil.rmtree(xdir)
R.generate_fixture(str(xdir), 2, (1, 4, 4, 4), loss="xent", seed=2)
vox = R._fixture_voxels(7, 3, (2, 3, 4, 5))
out["fixture_7_3"] = vox.reshape(-1).tolist()
(here / "datastore.json").write_text(json.dumps(out))
print("wrote", here / "datastore.json")
