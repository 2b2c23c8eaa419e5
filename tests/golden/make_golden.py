"""Generate tests/golden/*.json / *.npz from the REFERENCE ITSELF.

Runs the unmodified reference library (oracle/_ref/libtpfuse_ref.so, compiled by
oracle/Makefile from /root/reference/proj/src) and freezes its outputs so the
GPU box — where /root/reference does not exist — can check against them.

    python tests/golden/make_golden.py      # in the build container

Fixtures:
  schedules.json  build_schedule(kind, n) for kind in {ring, pairwise, circular},
                  n = 1..8 (or the rejection message), ring_indices_ag/rs tables.
  cases.npz       small integer-data outputs of column_parallel_forward,
                  row_parallel_forward and tpsp_mlp_forward (square activation),
                  generated with the reference's verify_mlp recipe
                  (randint_fill + mix_seed, experiment.cpp:302-330).
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import Oracle, OracleError, Reference  # noqa: E402

# (T, kind, m, B, S, D, H) — SPEC acceptance C1 desk scale (B=2, S=64, D=32, H=64)
CASES = [(t, kind, m, 2, 64, 32, 64) for t in (1, 2, 4, 8) for kind in (0, 1, 2) for m in (1, 2)
         if not (kind != 0 and m > 1) and not (kind == 1 and t % 2 and t != 1)]


def main() -> None:
    R = Reference()
    O = Oracle()
    sched = {"ring_indices_ag": {}, "ring_indices_rs": {}, "schedules": {}}
    for n in range(1, 9):
        sched["ring_indices_ag"][str(n)] = [[list(R.ring_indices(False, r, i, n)) for i in range(n)] for r in range(n)]
        sched["ring_indices_rs"][str(n)] = [[list(R.ring_indices(True, r, i, n)) for i in range(n)] for r in range(n)]
        for kind in (0, 1, 2):
            key = f"{kind}/{n}"
            try:
                sched["schedules"][key] = R.schedule(kind, n).tolist()
            except OracleError as e:
                sched["schedules"][key] = {"rejected": str(e)}
    sched["randint_fill_1_2_2_0_8_42"] = R.randint((1, 2, 2), 0, 8, 42).reshape(-1).tolist()
    with open(os.path.join(HERE, "schedules.json"), "w") as f:
        json.dump(sched, f, indent=None, separators=(",", ":"))

    arrays = {}
    for idx, (t, kind, m, b, s, d, h) in enumerate(CASES):
        seed = idx % 5
        x = R.randint((b, s, d), 0, 5, O.mix_seed(seed, 0))
        up = R.randint_matrix(d, h, -2, 2, O.mix_seed(seed, 1))
        down = R.randint_matrix(h, d, -2, 2, O.mix_seed(seed, 2))
        x2 = R.randint((b, s, d), 0, 5, O.mix_seed(seed, 3))
        w2 = R.randint_matrix(d, d, -2, 2, O.mix_seed(seed, 4))
        tag = f"t{t}_k{kind}_m{m}"
        arrays[f"{tag}/x"] = x
        arrays[f"{tag}/up"] = up
        arrays[f"{tag}/down"] = down
        arrays[f"{tag}/x2"] = x2
        arrays[f"{tag}/w2"] = w2
        arrays[f"{tag}/mlp"] = R.mlp_square(t, kind, m, x, up, down)
        arrays[f"{tag}/col"] = R.column_parallel(t, m, x, up)
        arrays[f"{tag}/row"] = R.row_parallel(t, kind, m, x2, w2)
    np.savez_compressed(os.path.join(HERE, "cases.npz"), **arrays)
    print(f"wrote {len(sched['schedules'])} schedules, {len(CASES)} cases")


if __name__ == "__main__":
    main()
