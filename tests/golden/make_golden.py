#!/usr/bin/env python
"""Regenerate tests/golden/ from the reference itself (oracle/_ref = the reference headers
compiled unmodified). Run here, where /root/reference exists:

    make -C oracle ref && python tests/golden/make_golden.py

The fixtures pin the C restatement (oracle/liboracle.so) and the CUDA engine on the GPU box,
where the reference tree is absent.
"""
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle.oracle import Oracle  # noqa: E402

OUT = Path(__file__).resolve().parent


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        if a.dtype.names:  # structured (gates / record entries): hash fields, never padding
            for f in a.dtype.names:
                h.update(np.ascontiguousarray(a[f]).tobytes())
        else:
            h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


RUNS = [  # (n, depth, circuit seed, p, run seed)
    (1, 3, 5, 1.0, 2), (2, 6, 7, 0.5, 3), (5, 10, 11, 1.0, 4), (63, 20, 1, 0.7, 7), (64, 25, 2, 1.0, 8),
    (65, 30, 3, 0.9, 9), (130, 40, 4, 0.6, 10), (200, 12, 31, 0.5, 0), (1000, 100, 42, 1.0, 7),
]
SAMPLES = [  # (n, depth, seed, p, shots, sample seed)
    (6, 10, 91, 1.0, 64, 1234), (6, 10, 91, 1.0, 128, 1234), (8, 12, 5, 0.7, 500, 42), (20, 30, 3, 1.0, 1000, 9),
]


def main():
    ref = Oracle("reference")
    fixtures, arrays = {"runs": [], "samples": []}, {}
    for i, (n, d, cs, p, rs) in enumerate(RUNS):
        g = ref.generate_random(n, d, cs, p)
        x, z, s, rec, rep = ref.run_single_shot(n, g, rs)
        item = {"n": n, "depth": d, "circuit_seed": cs, "p": p, "run_seed": rs, "gates": int(len(g)),
                "gates_sha256": digest(g), "tableau_sha256": digest(x, z, s), "record_sha256": digest(rec),
                "probabilistic": int(rep.probabilistic_count)}
        if n <= 200:
            arrays[f"run{i}_x"], arrays[f"run{i}_z"], arrays[f"run{i}_s"] = x, z, s
            arrays[f"run{i}_rec"] = rec
            item["arrays"] = f"run{i}"
        fixtures["runs"].append(item)
    for i, (n, d, cs, p, shots, ss) in enumerate(SAMPLES):
        g = ref.generate_random(n, d, cs, p)
        meas, words, _ = ref.sample(n, g, shots, ss)
        arrays[f"sample{i}_measured"], arrays[f"sample{i}_words"] = meas, words
        fixtures["samples"].append({"n": n, "depth": d, "circuit_seed": cs, "p": p, "shots": shots,
                                    "seed": ss, "arrays": f"sample{i}"})
    # transposes of a random tableau (test_tableau.cpp:165-178 analogue)
    rng = np.random.default_rng(42)
    for n in (1, 63, 64, 65, 100):
        k = (n + 63) // 64
        x, z, s = ref.basis_state(n)
        c = ref.generate_random(n, 8, 100 + n, 0.0)
        ref.apply_window  # scramble through the reference scheduler + windows
        sg, off, fl = ref.schedule(n, c, 0)
        for w in range(len(fl)):
            ref.apply_window(n, 0, x, z, s, sg[off[w]:off[w + 1]])
        arrays[f"tr{n}_cm_x"], arrays[f"tr{n}_cm_z"] = x.copy(), z.copy()
        ref.transpose(n, 0, x, z)
        arrays[f"tr{n}_rm_x"], arrays[f"tr{n}_rm_z"], arrays[f"tr{n}_s"] = x, z, s
        del k
    np.savez_compressed(OUT / "golden.npz", **arrays)
    (OUT / "golden.json").write_text(json.dumps(fixtures, indent=1) + "\n")
    print(f"wrote {len(arrays)} arrays, {len(fixtures['runs'])} runs, {len(fixtures['samples'])} samples")


if __name__ == "__main__":
    main()
