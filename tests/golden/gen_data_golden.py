"""Golden outputs of the reference's data module (pkg/src/svdrec/data.py)
on seeded inputs (tests/golden/inputs.py).  Run in the build container,
where /root/reference is importable; writes tests/golden/data.npz.

python tests/golden/gen_data_golden.py
"""
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
import inputs  # noqa: E402
from svdrec import data as D  # noqa: E402


def ds_arrays(ds):
    s = ds.samples
    return (np.array([x.user for x in s], np.int64), np.array([x.item for x in s], np.int64),
            np.array([x.rating for x in s], np.float64))


def main():
    out = {}
    with tempfile.TemporaryDirectory() as td:
        cases = {"csv": (inputs.ratings_csv_text(1, 3000), None),
                 "tsv": (inputs.ratings_csv_text(2, 800, delimiter="\t", header=False),
                         D.CsvSchema(delimiter="\t", has_header=False))}
        for name, (text, schema) in cases.items():
            p = Path(td) / f"{name}.txt"
            p.write_text(text)
            ds = D.load_ratings_csv(p, schema)
            u, i, r = ds_arrays(ds)
            out[f"{name}_users"], out[f"{name}_items"], out[f"{name}_ratings"] = u, i, r
            out[f"{name}_uids"] = np.array(list(ds.user_index.keys()))
            out[f"{name}_iids"] = np.array(list(ds.item_index.keys()))
            out[f"{name}_meta"] = np.array([ds.rating_min, ds.rating_max, ds.n_duplicates], np.float64)
            for mc in (2, 5):
                pr = D.prune_min_degree(ds, mc)
                u, i, r = ds_arrays(pr)
                out[f"{name}_prune{mc}"] = np.stack([u, i]).astype(np.int64)
                out[f"{name}_prune{mc}_r"] = r
                out[f"{name}_prune{mc}_uids"] = np.array(list(pr.user_index.keys()))
            A, val, test = D.split(ds, D.SplitSpec(0.8, 0.1, 0.1, seed=3))
            out[f"{name}_split_train"] = A.to_dense()
            out[f"{name}_split_val"] = np.array([tuple(s) for s in val], np.float64)
            out[f"{name}_split_test"] = np.array([tuple(s) for s in test], np.float64)
        p = Path(td) / "m.mtx"
        p.write_text(inputs.matrix_market_text(4, 30, 20, 90))
        out["mtx_dense"] = D.load_matrix_market(p).to_dense()
        p.write_text(inputs.matrix_market_text(5, 12, 9, 20, field="integer"))
        out["mtx_int_dense"] = D.load_matrix_market(p).to_dense()
    np.savez_compressed(HERE / "data.npz", **out)
    print("wrote", HERE / "data.npz", len(out), "arrays")


if __name__ == "__main__":
    main()
