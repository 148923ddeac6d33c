"""Record sinks and the synthetic dataset (src/taucorr/dataio.py:32-118, 200-219).

Host-side consumers of the device record stream, byte-compatible with the
reference: TSV lines and the raw 48-byte CELL_DTYPE binary stream with the
all-ones n_d sentinel for an undefined tau_b.
"""

from __future__ import annotations

import numpy as np

from .engine import CELL_DTYPE, Dataset
from .errors import ParseError
from .result import derive_taus
from .workloads import synth_ranks

ND_SENTINEL = np.uint64(0xFFFFFFFFFFFFFFFF)


def _fmt(x: float) -> str:
    return repr(float(x))


def render_tsv_lines(records: np.ndarray, labels, n: int, tau_b_valid: bool = True):
    """label_i, label_j, tau_b, tau_a, n_d, n1, n2, n3 per record (dataio.py:40-53)."""
    tau_a, tau_b = derive_taus(records["numerator"], records["n1"], records["n2"], n, tau_b_valid)
    ii, jj = records["i"], records["j"]
    nd, n1, n2, n3 = records["n_d"], records["n1"], records["n2"], records["n3"]
    for k in range(records.shape[0]):
        yield (f"{labels[ii[k]]}\t{labels[jj[k]]}\t{_fmt(tau_b[k])}\t{_fmt(tau_a[k])}"
               f"\t{nd[k]}\t{n1[k]}\t{n2[k]}\t{n3[k]}\n")


class TsvWriter:
    def __init__(self, stream, labels, n: int, kernel: str = "sorted", skip_diagonal: bool = False):
        self._stream = stream
        self._labels = list(labels)
        self._n = n
        self._tau_b_valid = kernel != "naive"
        self._skip_diagonal = skip_diagonal

    def __call__(self, records: np.ndarray) -> None:
        if self._skip_diagonal:
            records = records[records["i"] != records["j"]]
        self._stream.write("".join(render_tsv_lines(records, self._labels, self._n, self._tau_b_valid)))


class BinaryWriter:
    """Raw CELL_DTYPE records; n_d = all-ones where tau_b is undefined (dataio.py:74-93)."""

    def __init__(self, stream, n: int, kernel: str = "sorted", skip_diagonal: bool = False):
        self._stream = stream
        self._n = n
        self._tau_b_valid = kernel != "naive"
        self._skip_diagonal = skip_diagonal

    def __call__(self, records: np.ndarray) -> None:
        if self._skip_diagonal:
            records = records[records["i"] != records["j"]]
        out = records.copy()
        n0 = self._n * (self._n - 1) // 2
        if self._tau_b_valid:
            undefined = (out["n1"] >= n0) | (out["n2"] >= n0)
        else:
            undefined = np.ones(out.shape[0], dtype=bool)
        out["n_d"][undefined] = ND_SENTINEL
        self._stream.write(out.tobytes())


def read_binary(source, n: int):
    """(records, tau_a, tau_b) from a binary stream (dataio.py:96-118)."""
    if hasattr(source, "read"):
        raw = source.read()
    else:
        with open(source, "rb") as fh:
            raw = fh.read()
    if len(raw) % CELL_DTYPE.itemsize:
        raise ParseError(f"binary stream length {len(raw)} is not a multiple of {CELL_DTYPE.itemsize}")
    records = np.frombuffer(raw, dtype=CELL_DTYPE).copy()
    undefined = records["n_d"] == ND_SENTINEL
    records["n_d"][undefined] = 0
    tau_a, tau_b = derive_taus(records["numerator"], records["n1"], records["n2"], n)
    return records, tau_a, np.where(undefined, np.nan, tau_b)


def synth_dataset(m: int, n: int, tie_fraction: float = 0.0, seed: int = 0) -> Dataset:
    """Deterministic dense-rank dataset, same draws as dataio.py:200-219."""
    from .errors import InvalidInputError

    try:
        ranks = synth_ranks(m, n, tie_fraction, seed)
    except ValueError as exc:
        raise InvalidInputError(str(exc)) from None
    return Dataset(labels=[f"V{k}" for k in range(m)], ranks=ranks)
