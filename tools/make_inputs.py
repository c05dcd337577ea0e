"""Seeded synthetic inputs of the BASELINE configs as .ffsoa files plus a manifest
("fp64 SoA binary plus a manifest (seed, N, sha256)").

    python tools/make_inputs.py --workload c2 --out /tmp/inputs [--events N] [--rank R]

Writes <workload>[.rR].ffsoa (the generator's columns, exactly what bench.py samples for
that rank) and <workload>[.rR].json = {workload, model, seed, n, columns, sha256, generator}.
`bench.py --inputs DIR` loads them instead of sampling."""
import argparse
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2003_12875_b200 as fb
from paper_2003_12875_b200 import configs


def shard_seed(w, rank):  # the same seeds as bench.py
    return w.data_seed if rank == 0 else w.data_seed + 100003 * rank


def file_name(w, rank):
    return w.name + (f".r{rank}" if rank else "")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--out", required=True)
    ap.add_argument("--events", type=int, default=0)
    ap.add_argument("--rank", type=int, default=0)
    a = ap.parse_args()
    key = a.workload.lower()
    w = configs.BY_INDEX[int(key[1]) - 1] if key in ("c1", "c2", "c3", "c4", "c5") else configs.WORKLOADS[a.workload]
    n = a.events or w.n_events
    seed = shard_seed(w, a.rank)
    cols, eff = fb.sample_host(fb.Model.from_string(w.text), n, seed)
    os.makedirs(a.out, exist_ok=True)
    path = os.path.join(a.out, file_name(w, a.rank) + ".ffsoa")
    fb.write_soa(path, cols)
    h = hashlib.sha256()
    with open(path, "rb") as fh:
        for chunk in iter(lambda: fh.read(1 << 24), b""):
            h.update(chunk)
    manifest = {"workload": w.name, "model": w.text, "seed": seed, "n": n, "columns": list(cols),
                "sha256": h.hexdigest(), "file": os.path.basename(path),
                "generator": "reference Rng (xoshiro256++ / splitmix64) restated, csrc/sampler.cpp; "
                             "accept/reject efficiency %.6f" % eff}
    with open(os.path.join(a.out, file_name(w, a.rank) + ".json"), "w") as fh:
        json.dump(manifest, fh, indent=1)
    print(json.dumps({k: v for k, v in manifest.items() if k != "model"}))


if __name__ == "__main__":
    main()
