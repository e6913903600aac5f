"""Ingest bench: load_ratings_csv -> prune_min_degree -> split on a seeded
delimited file, this package vs the reference's data module (imported from
/root/reference when present, else this package's row-by-row exact path,
which restates it).  Host-side; prints one JSON line.

python tools/bench_data.py [--rows N]
"""
import argparse
import json
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests" / "golden"))


def run(mod, path, reps=1):
    best = None
    for _ in range(reps):
        t = time.perf_counter()
        ds = mod.load_ratings_csv(path)
        t1 = time.perf_counter()
        pr = mod.prune_min_degree(ds, 5)
        t2 = time.perf_counter()
        A, val, test = mod.split(pr, mod.SplitSpec(0.9, 0.05, 0.05, seed=0))
        t3 = time.perf_counter()
        cur = (t1 - t, t2 - t1, t3 - t2, t3 - t, A.nnz, len(val), len(test))
        best = cur if best is None or cur[3] < best[3] else best
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=2_000_000)
    args = ap.parse_args()
    import inputs
    from paper_2009_02251_b200 import data as ours
    ref_kind = "reference (svdrec.data)"
    try:
        sys.path.insert(0, "/root/reference/pkg/src")
        from svdrec import data as ref
    except Exception:
        ref, ref_kind = None, "port (row-by-row exact path)"
    with tempfile.TemporaryDirectory() as td:
        p = Path(td) / "ratings.csv"
        p.write_text(inputs.ratings_csv_text(3, args.rows, nusers=max(50, args.rows // 40),
                                             nitems=max(40, args.rows // 200), dup_frac=0.01))
        o = run(ours, p, reps=2)
        if ref is not None:
            r = run(ref, p)
        else:
            class Exact:
                load_ratings_csv = staticmethod(lambda q: ours._load_csv_exact(Path(q), ours.CsvSchema()))
                prune_min_degree = staticmethod(ours.prune_min_degree)
                split = staticmethod(ours.split)
                SplitSpec = ours.SplitSpec
            r = run(Exact, p)
    assert o[4:] == r[4:], (o, r)
    print(json.dumps({"metric": "ingest time (s): load_ratings_csv + prune_min_degree(5) + split", "rows": args.rows,
                      "ours_s": round(o[3], 3), "ours_phases_s": [round(x, 3) for x in o[:3]],
                      "reference_s": round(r[3], 3), "reference_phases_s": [round(x, 3) for x in r[:3]],
                      "reference_kind": ref_kind, "speedup": round(r[3] / o[3], 2),
                      "same_split_sizes": True, "train_nnz": o[4]}))


if __name__ == "__main__":
    main()
