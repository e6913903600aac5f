"""Dataset ingest (paper_2009_02251_b200.data): parity with the reference's
data module on seeded inputs (tests/golden/data.npz, produced by
tests/golden/gen_data_golden.py running the reference itself) and the
module's behavioural contract.  CPU only."""
import sys
from pathlib import Path

import numpy as np
import pytest

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE / "golden"))

import inputs  # noqa: E402
from paper_2009_02251_b200 import data as D  # noqa: E402
from paper_2009_02251_b200 import SparseRatings  # noqa: E402

G = np.load(HERE / "golden" / "data.npz")


def _load(tmp_path, name):
    if name == "csv":
        p = tmp_path / "r.csv"
        p.write_text(inputs.ratings_csv_text(1, 3000))
        return D.load_ratings_csv(p)
    p = tmp_path / "r.tsv"
    p.write_text(inputs.ratings_csv_text(2, 800, delimiter="\t", header=False))
    return D.load_ratings_csv(p, D.CsvSchema(delimiter="\t", has_header=False))


@pytest.mark.parametrize("name", ["csv", "tsv"])
def test_loader_matches_reference(tmp_path, name):
    ds = _load(tmp_path, name)
    u, i, r = ds.arrays()
    np.testing.assert_array_equal(u, G[f"{name}_users"])
    np.testing.assert_array_equal(i, G[f"{name}_items"])
    np.testing.assert_array_equal(r, G[f"{name}_ratings"])
    assert list(ds.user_index) == G[f"{name}_uids"].tolist()
    assert list(ds.item_index) == G[f"{name}_iids"].tolist()
    assert [ds.rating_min, ds.rating_max, ds.n_duplicates] == G[f"{name}_meta"].tolist()
    assert ds.samples[0] == D.RatingSample(int(u[0]), int(i[0]), float(r[0]))


@pytest.mark.parametrize("name", ["csv", "tsv"])
@pytest.mark.parametrize("mc", [2, 5])
def test_prune_matches_reference(tmp_path, name, mc):
    pr = D.prune_min_degree(_load(tmp_path, name), mc)
    u, i, r = pr.arrays()
    np.testing.assert_array_equal(np.stack([u, i]), G[f"{name}_prune{mc}"])
    np.testing.assert_array_equal(r, G[f"{name}_prune{mc}_r"])
    assert list(pr.user_index) == G[f"{name}_prune{mc}_uids"].tolist()


@pytest.mark.parametrize("name", ["csv", "tsv"])
def test_split_matches_reference(tmp_path, name):
    A, val, test = D.split(_load(tmp_path, name), D.SplitSpec(0.8, 0.1, 0.1, seed=3))
    np.testing.assert_array_equal(A.to_dense(), G[f"{name}_split_train"])
    np.testing.assert_array_equal(np.array([tuple(s) for s in val], np.float64), G[f"{name}_split_val"])
    np.testing.assert_array_equal(np.array([tuple(s) for s in test], np.float64), G[f"{name}_split_test"])
    assert isinstance(val, list) and isinstance(val[0], D.RatingSample)


def test_matrix_market_matches_reference(tmp_path):
    p = tmp_path / "m.mtx"
    p.write_text(inputs.matrix_market_text(4, 30, 20, 90))
    np.testing.assert_array_equal(D.load_matrix_market(p).to_dense(), G["mtx_dense"])
    p.write_text(inputs.matrix_market_text(5, 12, 9, 20, field="integer"))
    np.testing.assert_array_equal(D.load_matrix_market(p).to_dense(), G["mtx_int_dense"])


def test_matrix_market_round_trip(tmp_path):
    p = tmp_path / "m.mtx"
    p.write_text(inputs.matrix_market_text(6, 25, 17, 60))
    A = D.load_matrix_market(p)
    q = tmp_path / "copy.mtx"
    D.save_matrix_market(q, A)
    B = D.load_matrix_market(q)
    np.testing.assert_array_equal(A.to_dense(), B.to_dense())
    assert (A.rating_min, A.rating_max) == (B.rating_min, B.rating_max)


@pytest.mark.parametrize("text, where", [
    ("u,i,r\na,b,4\nc,d\n", "line 3"),            # short row
    ("u,i,r\na,b,4\nc,d,x\n", "line 3"),          # bad rating
    ("u,i,r\na,b,inf\n", "line 2"),               # non-finite
    ("u,i,r\na, ,4\n", "line 2"),                 # empty identifier
])
def test_malformed_rows_name_the_line(tmp_path, text, where):
    p = tmp_path / "bad.csv"
    p.write_text(text)
    with pytest.raises(D.DataFormatError, match=where):
        D.load_ratings_csv(p)


def test_empty_and_blank_files(tmp_path):
    p = tmp_path / "e.csv"
    p.write_text("u,i,r\n\n   \n")
    with pytest.raises(D.EmptyDatasetError):
        D.load_ratings_csv(p)
    q = tmp_path / "b.csv"
    q.write_text("u,i,r\na,b,4\n\n  \nc,d,2\n")
    ds = D.load_ratings_csv(q)
    assert ds.nnz == 2 and ds.m == 2 and ds.n == 2


def test_duplicates_keep_last_and_count(tmp_path):
    p = tmp_path / "d.csv"
    p.write_text("u,i,r\na,x,1\nb,y,2\na,x,3\na,x,5\n")
    ds = D.load_ratings_csv(p)
    assert ds.n_duplicates == 2
    assert ds.samples == [D.RatingSample(0, 0, 5.0), D.RatingSample(1, 1, 2.0)]


def test_extra_fields_are_allowed(tmp_path):
    p = tmp_path / "x.csv"
    p.write_text("u,i,r\na,b,4,extra\nc,d,2\n")  # ragged but long enough
    ds = D.load_ratings_csv(p)
    assert ds.nnz == 2


def test_schema_and_spec_validation():
    with pytest.raises(ValueError):
        D.CsvSchema(user_col=1, item_col=1)
    with pytest.raises(ValueError):
        D.CsvSchema(rating_col=-1)
    with pytest.raises(ValueError):
        D.SplitSpec(0.9, 0.1, 0.0)
    with pytest.raises(ValueError):
        D.SplitSpec(0.5, 0.2, 0.2)


def test_prune_fixed_point_identity_and_errors(tmp_path):
    ds = _load(tmp_path, "csv")
    assert D.prune_min_degree(ds, 1) is ds
    with pytest.raises(D.EmptyDatasetError):
        D.prune_min_degree(ds, 10 ** 6)
    with pytest.raises(ValueError):
        D.prune_min_degree(ds, 0)
    pr = D.prune_min_degree(ds, 5)
    u, i, _ = pr.arrays()
    assert np.bincount(u).min() >= 5 and np.bincount(i).min() >= 5


def test_split_union_and_zero_part(tmp_path):
    ds = _load(tmp_path, "csv")
    A, val, test = D.split(ds, D.SplitSpec(seed=9))
    assert A.nnz + len(val) + len(test) == ds.nnz
    assert A.shape == (ds.m, ds.n)
    tiny = D.RatingsDataset({"a": 0}, {"x": 0}, [D.RatingSample(0, 0, 1.0)], 1.0, 1.0)
    with pytest.raises(ValueError):
        D.split(tiny, D.SplitSpec())


def test_matrix_market_errors(tmp_path):
    p = tmp_path / "bad.mtx"
    for text, exc in [("no banner\n1 1 1\n1 1 1\n", D.DataFormatError),
                      ("%%MatrixMarket matrix array real general\n1 1\n1\n", D.DataFormatError),
                      ("%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 1 1\n", D.DataFormatError),
                      ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n", D.DataFormatError),
                      ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n", D.DataFormatError),
                      ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n1 1 2\n", ValueError)]:
        p.write_text(text)
        with pytest.raises(exc):
            D.load_matrix_market(p)


def test_manifest_and_dataset_to_sparse(tmp_path):
    ds = _load(tmp_path, "tsv")
    A = D.dataset_to_sparse(ds)
    assert A.nnz == ds.nnz and A.shape == (ds.m, ds.n)
    spec = D.SplitSpec(0.8, 0.1, 0.1, seed=2)
    D.write_split_manifest(tmp_path / "man.txt", spec, (8, 1, 1))
    text = (tmp_path / "man.txt").read_text()
    assert "seed = 2" in text and "total = 10" in text


def test_matrix_market_round_trip_random_doubles(tmp_path):
    """Lossless round trip for arbitrary doubles (the fast parser must round
    like float(); pandas' default converter changed ~15 % of such values)."""
    from scipy import sparse as sp
    rng = np.random.default_rng(11)
    m, n, nnz = 120, 90, 6000
    flat = rng.choice(m * n, nnz, replace=False)
    vals = rng.uniform(0.5, 5.0, nnz)
    M = sp.csr_matrix((vals, (flat // n, flat % n)), shape=(m, n))
    A = SparseRatings(M, 0.5, 5.0)
    p = tmp_path / "r.mtx"
    D.save_matrix_market(p, A)
    B = D.load_matrix_market(p)
    assert np.array_equal(A.to_dense(), B.to_dense())


def test_csv_ratings_parse_like_float(tmp_path):
    rng = np.random.default_rng(12)
    vals = rng.uniform(0.5, 5.0, 4000)
    p = tmp_path / "r.csv"
    p.write_text("u,i,r\n" + "".join(f"u{k},i{k % 97},{repr(float(v))}\n" for k, v in enumerate(vals)))
    ds = D.load_ratings_csv(p)
    got = np.array([s[2] for s in ds.samples])
    assert np.array_equal(np.sort(got), np.sort(vals))
