"""Rating-dataset ingest: loading, pruning, splitting (the callers before the
factorisation path).

Same public names, arguments, results and errors as the reference's
``svdrec.data`` (pkg/src/svdrec/data.py).  The reference walks every row in
Python (csv.reader + dict lookups per rating); here every pass over the
ratings is vectorised: delimited files go through pandas' C parser,
identifiers are mapped to dense indices in first-appearance order with
``pandas.factorize``, duplicates are resolved with one sort, pruning is an
iterated ``bincount`` fixed point.  Whenever the fast path sees anything
irregular (short rows, unparsable fields, blank-but-not-empty lines...) the
file is re-read by the exact row-by-row path, so error types and messages
(``DataFormatError`` naming the line) are the reference's.
"""
from __future__ import annotations

import csv
from dataclasses import dataclass
from pathlib import Path
from typing import NamedTuple

import numpy as np

from .sparse import SparseRatings


class DataFormatError(ValueError):
    """Input file violates the expected format."""


class EmptyDatasetError(ValueError):
    """An operation would leave or found no ratings."""


class RatingSample(NamedTuple):
    """(user, item, rating) triple with dense indices."""

    user: int
    item: int
    rating: float


@dataclass(frozen=True)
class CsvSchema:
    """Column layout of a delimited ratings file (data.py:38-51)."""

    delimiter: str = ","
    user_col: int = 0
    item_col: int = 1
    rating_col: int = 2
    has_header: bool = True

    def __post_init__(self) -> None:
        cols = (self.user_col, self.item_col, self.rating_col)
        if len(set(cols)) != 3 or min(cols) < 0:
            raise ValueError("user, item, rating columns must be distinct and >= 0")


class SampleList(list):
    """A list of RatingSample that also carries the triples as arrays, so
    the GPU scoring path groups them without walking Python objects."""

    def __init__(self, users: np.ndarray, items: np.ndarray, ratings: np.ndarray):
        super().__init__(RatingSample(int(u), int(i), float(r))
                         for u, i, r in zip(users.tolist(), items.tolist(), ratings.tolist()))
        self.arrays = (users, items, ratings)


class RatingsDataset:
    """Ratings in dense-index form plus the raw-identifier mappings
    (data.py:54-75).  Holds the triples as arrays; ``samples`` is the list
    view of the reference's dataclass field."""

    def __init__(self, user_index: dict, item_index: dict, samples, rating_min: float, rating_max: float,
                 n_duplicates: int = 0):
        self.user_index = user_index
        self.item_index = item_index
        self.rating_min = rating_min
        self.rating_max = rating_max
        self.n_duplicates = n_duplicates
        self._samples = samples
        self._arr = samples.arrays if isinstance(samples, SampleList) else None

    @classmethod
    def _from_arrays(cls, user_index, item_index, users, items, ratings, n_duplicates=0):
        ds = cls(user_index, item_index, None, float(ratings.min()), float(ratings.max()), n_duplicates)
        ds._arr = (users, items, ratings)
        return ds

    @property
    def samples(self) -> list:
        if self._samples is None:
            self._samples = SampleList(*self._arr)
        return self._samples

    @samples.setter
    def samples(self, value) -> None:
        self._samples = value
        self._arr = value.arrays if isinstance(value, SampleList) else None

    def arrays(self) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        if self._arr is None:
            s = self._samples
            self._arr = (np.fromiter((x[0] for x in s), np.int64, len(s)),
                         np.fromiter((x[1] for x in s), np.int64, len(s)),
                         np.fromiter((x[2] for x in s), np.float64, len(s)))
        return self._arr

    @property
    def m(self) -> int:
        return len(self.user_index)

    @property
    def n(self) -> int:
        return len(self.item_index)

    @property
    def nnz(self) -> int:
        return len(self._samples) if self._samples is not None else int(self._arr[0].size)


@dataclass(frozen=True)
class SplitSpec:
    """Train/validation/test fractions plus the shuffle seed (data.py:78-91)."""

    train: float = 0.9
    validation: float = 0.05
    test: float = 0.05
    seed: int = 0

    def __post_init__(self) -> None:
        parts = (self.train, self.validation, self.test)
        if min(parts) <= 0.0:
            raise ValueError("all three fractions must be positive")
        if abs(sum(parts) - 1.0) > 1e-12:
            raise ValueError(f"fractions must sum to 1, got {sum(parts)}")


# ---------------------------------------------------------------------------
# delimited files

def _dedupe(users: np.ndarray, items: np.ndarray, ratings: np.ndarray, n_items: int):
    """Pairs in order of first appearance, each with its last value; the
    number of repeated occurrences (data.py:94-148 semantics)."""
    key = users * max(n_items, 1) + items
    order = np.argsort(key, kind="stable")
    ks = key[order]
    start = np.r_[True, ks[1:] != ks[:-1]]
    end = np.r_[ks[1:] != ks[:-1], True]
    first = order[start]  # earliest occurrence of each pair
    last = order[end]     # latest occurrence of each pair
    pos = np.argsort(first, kind="stable")
    keep_first, keep_last = first[pos], last[pos]
    return users[keep_first], items[keep_first], ratings[keep_last], int(key.size - keep_first.size)


def _load_csv_exact(path: Path, schema: CsvSchema) -> RatingsDataset:
    """Row-by-row restatement of the reference loader (used for error
    reporting and as the fallback of the vectorised path)."""
    need = max(schema.user_col, schema.item_col, schema.rating_col) + 1
    user_index: dict[str, int] = {}
    item_index: dict[str, int] = {}
    cells: dict[tuple[int, int], float] = {}
    n_dup = 0
    with path.open(newline="") as handle:
        for lineno, row in enumerate(csv.reader(handle, delimiter=schema.delimiter), start=1):
            if lineno == 1 and schema.has_header:
                continue
            if not row or (len(row) == 1 and not row[0].strip()):
                continue
            if len(row) < need:
                raise DataFormatError(f"{path}: line {lineno}: expected at least {need} fields, got {len(row)}")
            raw_user, raw_item = row[schema.user_col].strip(), row[schema.item_col].strip()
            try:
                rating = float(row[schema.rating_col])
            except ValueError as exc:
                raise DataFormatError(f"{path}: line {lineno}: bad rating {row[schema.rating_col]!r}") from exc
            if not np.isfinite(rating):
                raise DataFormatError(f"{path}: line {lineno}: non-finite rating")
            if not raw_user or not raw_item:
                raise DataFormatError(f"{path}: line {lineno}: empty identifier")
            u = user_index.setdefault(raw_user, len(user_index))
            i = item_index.setdefault(raw_item, len(item_index))
            if (u, i) in cells:
                n_dup += 1
            cells[(u, i)] = rating
    if not cells:
        raise EmptyDatasetError(f"{path}: no ratings found")
    n = len(cells)
    users = np.fromiter((k[0] for k in cells), np.int64, n)
    items = np.fromiter((k[1] for k in cells), np.int64, n)
    vals = np.fromiter(cells.values(), np.float64, n)
    return RatingsDataset._from_arrays(user_index, item_index, users, items, vals, n_dup)


def _codes(raw) -> tuple[np.ndarray, list]:
    """Dense codes in first-appearance order of the *stripped* identifiers
    (factorise the raw strings, strip only the distinct values)."""
    import pandas as pd
    code, uniq = pd.factorize(raw, sort=False)
    names = [str(x) for x in uniq.tolist()]
    stripped = [x.strip() for x in names]
    if stripped != names:  # whitespace variants of one identifier merge
        code2, uniq2 = pd.factorize(np.asarray(stripped, dtype=object), sort=False)
        return code2[code].astype(np.int64), [str(x) for x in uniq2.tolist()]
    return code.astype(np.int64), names


def _load_csv_fast(path: Path, schema: CsvSchema) -> RatingsDataset | None:
    """Vectorised loader; None when the file needs the exact path."""
    try:
        import pandas as pd
    except ImportError:
        return None
    need = max(schema.user_col, schema.item_col, schema.rating_col) + 1
    try:
        # round_trip: the C parser's default float converter is not always
        # correctly rounded; the reference parses with float()
        df = pd.read_csv(path, float_precision="round_trip", sep=schema.delimiter, header=None,
                         skiprows=1 if schema.has_header else 0,
                         usecols=[schema.user_col, schema.item_col, schema.rating_col],
                         dtype={schema.user_col: str, schema.item_col: str, schema.rating_col: np.float64},
                         keep_default_na=False, na_filter=False, skip_blank_lines=True, engine="c",
                         quoting=csv.QUOTE_MINIMAL)
    except Exception:  # ragged rows, unparsable ratings, empty file: the exact path decides
        return None
    if df.shape[0] == 0:
        return None
    raw_u = df[schema.user_col].to_numpy(dtype=object)
    raw_i = df[schema.item_col].to_numpy(dtype=object)
    ratings = df[schema.rating_col].to_numpy(dtype=np.float64)
    if not np.all(np.isfinite(ratings)):
        return None
    ucode, unames = _codes(raw_u)
    icode, inames = _codes(raw_i)
    if "" in unames or "" in inames:
        return None  # empty identifier: reported with its line by the exact path
    users, items, vals, n_dup = _dedupe(ucode, icode, ratings, len(inames))
    return RatingsDataset._from_arrays({k: j for j, k in enumerate(unames)}, {k: j for j, k in enumerate(inames)},
                                       users, items, vals, n_dup)


def load_ratings_csv(path: str | Path, schema: CsvSchema | None = None) -> RatingsDataset:
    """Read a delimited ratings file into dense-index form (data.py:94-148).

    Duplicate (user, item) pairs keep the last value seen and are counted in
    ``n_duplicates``; a malformed row raises DataFormatError naming the line;
    a file without data rows raises EmptyDatasetError.
    """
    schema = schema or CsvSchema()
    path = Path(path)
    ds = _load_csv_fast(path, schema)
    return ds if ds is not None else _load_csv_exact(path, schema)


def prune_min_degree(ds: RatingsDataset, min_count: int) -> RatingsDataset:
    """Drop users / items with fewer than ``min_count`` ratings, iterated to
    a fixed point; survivors reindexed densely in order (data.py:151-197)."""
    if min_count < 1:
        raise ValueError("min_count must be at least 1")
    users, items, vals = ds.arrays()
    keep = np.ones(users.size, dtype=bool)
    while True:
        ud = np.bincount(users[keep], minlength=ds.m)
        idg = np.bincount(items[keep], minlength=ds.n)
        nk = keep & (ud[users] >= min_count) & (idg[items] >= min_count)
        if nk.sum() == keep.sum():
            break
        keep = nk
        if not keep.any():
            raise EmptyDatasetError(f"pruning at min_count={min_count} removed everything")
    if keep.all():
        return ds
    u, i, v = users[keep], items[keep], vals[keep]
    live_u, new_u = np.unique(u, return_inverse=True)
    live_i, new_i = np.unique(i, return_inverse=True)
    inv_user = {v_: k for k, v_ in ds.user_index.items()}
    inv_item = {v_: k for k, v_ in ds.item_index.items()}
    return RatingsDataset._from_arrays({inv_user[int(o)]: j for j, o in enumerate(live_u.tolist())},
                                       {inv_item[int(o)]: j for j, o in enumerate(live_i.tolist())},
                                       new_u.astype(np.int64), new_i.astype(np.int64), v, ds.n_duplicates)


def split(ds: RatingsDataset, spec: SplitSpec):
    """Seeded shuffle into a train matrix plus validation and test lists
    (data.py:200-232).  The train matrix keeps the dataset's full shape."""
    total = ds.nnz
    n_val = round(spec.validation * total)
    n_test = round(spec.test * total)
    n_train = total - n_val - n_test
    if min(n_train, n_val, n_test) <= 0:
        raise ValueError(f"split of {total} samples gives sizes ({n_train}, {n_val}, {n_test}); "
                         "every part must be nonempty")
    order = np.random.default_rng(spec.seed).permutation(total)
    users, items, vals = ds.arrays()
    tr, va, te = order[:n_train], order[n_train:n_train + n_val], order[n_train + n_val:]
    matrix = SparseRatings.from_coo(users[tr], items[tr], vals[tr], shape=(ds.m, ds.n),
                                    bounds=(ds.rating_min, ds.rating_max))
    return matrix, SampleList(users[va], items[va], vals[va]), SampleList(users[te], items[te], vals[te])


# ---------------------------------------------------------------------------
# Matrix Market

def _mm_header(path: Path, lines):
    banner = next(lines, "")
    if not banner.startswith("%%MatrixMarket"):
        raise DataFormatError(f"{path}: missing MatrixMarket banner")
    fields = banner.strip().split()
    if len(fields) != 5:
        raise DataFormatError(f"{path}: malformed banner: {banner.strip()!r}")
    _, obj, fmt, field, symmetry = (f.lower() for f in fields)
    if obj != "matrix" or fmt != "coordinate":
        raise DataFormatError(f"{path}: only coordinate matrices are supported")
    if field not in ("real", "integer"):
        raise DataFormatError(f"{path}: unsupported field type {field!r}")
    if symmetry != "general":
        raise DataFormatError(f"{path}: unsupported symmetry {symmetry!r}")


def _load_mm_exact(path: Path) -> SparseRatings:
    with path.open() as handle:
        it = iter(handle)
        _mm_header(path, it)
        lineno = 1
        size_line = None
        for line in it:
            lineno += 1
            s = line.strip()
            if not s or s.startswith("%"):
                continue
            size_line = s
            break
        if size_line is None:
            raise DataFormatError(f"{path}: missing size line")
        parts = size_line.split()
        if len(parts) != 3:
            raise DataFormatError(f"{path}: line {lineno}: bad size line")
        try:
            m, n, nnz = (int(p) for p in parts)
        except ValueError as exc:
            raise DataFormatError(f"{path}: line {lineno}: bad size line") from exc
        if m < 0 or n < 0 or nnz < 0:
            raise DataFormatError(f"{path}: line {lineno}: negative dimension")
        rows = np.empty(nnz, dtype=np.int64)
        cols = np.empty(nnz, dtype=np.int64)
        vals = np.empty(nnz, dtype=np.float64)
        count = 0
        for line in it:
            lineno += 1
            s = line.strip()
            if not s or s.startswith("%"):
                continue
            p = s.split()
            if len(p) != 3:
                raise DataFormatError(f"{path}: line {lineno}: expected 'row col value'")
            if count >= nnz:
                raise DataFormatError(f"{path}: more entries than declared ({nnz})")
            try:
                i, j, v = int(p[0]), int(p[1]), float(p[2])
            except ValueError as exc:
                raise DataFormatError(f"{path}: line {lineno}: bad entry") from exc
            if not (1 <= i <= m and 1 <= j <= n):
                raise DataFormatError(f"{path}: line {lineno}: entry ({i}, {j}) outside {m} x {n}")
            rows[count], cols[count], vals[count] = i - 1, j - 1, v
            count += 1
        if count != nnz:
            raise DataFormatError(f"{path}: declared {nnz} entries, found {count}")
    return SparseRatings.from_coo(rows, cols, vals, shape=(m, n))


def load_matrix_market(path: str | Path) -> SparseRatings:
    """Read a general real/integer Matrix Market coordinate file
    (data.py:235-308); rating bounds are the observed range."""
    path = Path(path)
    try:
        import pandas as pd
        with path.open() as handle:
            it = iter(handle)
            _mm_header(path, it)
            skip = 1
            size = None
            for line in it:
                skip += 1
                s = line.strip()
                if s and not s.startswith("%"):
                    size = s.split()
                    break
        if size is None or len(size) != 3:
            raise ValueError
        m, n, nnz = (int(x) for x in size)
        if min(m, n, nnz) < 0:
            raise ValueError
        df = pd.read_csv(path, float_precision="round_trip", sep=r"\s+", header=None, skiprows=skip, comment="%",
                         engine="c",
                         dtype={0: np.int64, 1: np.int64, 2: np.float64})
        if df.shape[1] != 3 or df.shape[0] != nnz:
            raise ValueError
        r = df.iloc[:, 0].to_numpy(np.int64)
        c = df.iloc[:, 1].to_numpy(np.int64)
        v = df.iloc[:, 2].to_numpy(np.float64)
        if nnz and (r.min() < 1 or r.max() > m or c.min() < 1 or c.max() > n):
            raise ValueError
        return SparseRatings.from_coo(r - 1, c - 1, v, shape=(m, n))
    except DataFormatError:
        raise
    except Exception:  # anything irregular: the exact path names the problem
        return _load_mm_exact(path)


def save_matrix_market(path: str | Path, ratings: SparseRatings) -> None:
    """Write ratings as a Matrix Market coordinate file (lossless round
    trip; data.py:311-319)."""
    path = Path(path)
    coo = ratings.matrix.tocoo()
    uniq, inv = np.unique(coo.data, return_inverse=True)
    reps = np.array([repr(float(x)) for x in uniq], dtype=object)
    with path.open("w") as handle:
        handle.write("%%MatrixMarket matrix coordinate real general\n")
        handle.write(f"{ratings.m} {ratings.n} {ratings.nnz}\n")
        rows = (coo.row + 1).astype(str)
        cols = (coo.col + 1).astype(str)
        for a in range(0, coo.nnz, 1 << 20):
            b = min(coo.nnz, a + (1 << 20))
            handle.write("".join(f"{i} {j} {v}\n" for i, j, v in zip(rows[a:b], cols[a:b], reps[inv[a:b]])))


def dataset_to_sparse(ds: RatingsDataset) -> SparseRatings:
    """All of a dataset's ratings as one matrix (data.py:322-329)."""
    u, i, v = ds.arrays()
    return SparseRatings.from_coo(u, i, v, shape=(ds.m, ds.n), bounds=(ds.rating_min, ds.rating_max))


def write_split_manifest(path: str | Path, spec: SplitSpec, counts: tuple[int, int, int]) -> None:
    """Record how a split was produced (data.py:332-348)."""
    n_train, n_val, n_test = counts
    lines = [f"seed = {spec.seed}", f"fractions = {spec.train},{spec.validation},{spec.test}",
             f"train = {n_train}", f"validation = {n_val}", f"test = {n_test}",
             f"total = {n_train + n_val + n_test}"]
    Path(path).write_text("\n".join(lines) + "\n")


__all__ = ["CsvSchema", "DataFormatError", "EmptyDatasetError", "RatingSample", "RatingsDataset", "SplitSpec",
           "dataset_to_sparse", "load_matrix_market", "load_ratings_csv", "prune_min_degree", "save_matrix_market",
           "split", "write_split_manifest"]
