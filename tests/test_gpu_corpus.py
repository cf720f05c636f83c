"""Corpus parsers on the GPU (hbp_load_lengths: raw-lengths, CSV) against
the reference's load_lengths (src/ingest.cpp:57-160) compiled in place
(oracle/_ref): same lengths, same first error, same message."""
import numpy as np
import pytest

from paper_2503_07680_b200 import abi

pytestmark = pytest.mark.gpu

RAW_CASES = [
    b"5\n7\n12\n", b"5\n7\n12", b"\n\n5\n \t\r\n7\r\n", b"  42  \n", b"+3\n", b"\x0b12\n", b"\x0c 9\n",
    b"9223372036854775807\n", b"1\n" * 5000,
    # errors (first failing line wins)
    b"5\nx\n", b"5\n7 8\n", b"0\n", b"-4\n", b"3\n-\n", b"+\n", b"12a\n", b"99999999999999999999\n",
    b"-9223372036854775808\n", b"1\n2\n0x10\n", b"", b"\n \n\t\n", b"5\n\x0b\n", b"1\n" * 3000 + b"2.5\n" + b"x\n",
]

CSV_CASES = [
    b"id,length\n1,5\n2,7\n", b"length\n5\n7", b"a, length ,b\n1, 12 ,x\n\n2,\t7\r,y\r\n", b"x,length,\n1,2,\n",
    b"length,x\n3,\n", b"length\r\n4\r\n",
    # errors
    b"", b"\n5\n", b"id,len\n1,2\n", b"id,length\n1\n", b"id,length\n1,\n", b"id,length\n1,abc\n",
    b"id,length\n1,0\n", b"id,length\n1,5 6\n", b"length\n", b"a,b,length\n1,2\n",
]


def _both(ctx, oracle, text, fmt):
    try:
        want = ("ok", oracle.load_lengths(text, fmt, "corpus.txt")[1].tolist())
    except Exception as e:  # noqa: BLE001
        want = (type(e).__name__, str(e))
    try:
        got = ("ok", ctx.load_lengths(text, fmt, "corpus.txt").tolist())
    except abi.ValidationError as e:
        got = ("ValidationError", str(e))
    return got, want


@pytest.mark.parametrize("i", range(len(RAW_CASES)))
def test_raw_lengths(ctx, reference, i):
    got, want = _both(ctx, reference, RAW_CASES[i], "raw-lengths")
    assert got == want


@pytest.mark.parametrize("i", range(len(CSV_CASES)))
def test_csv(ctx, reference, i):
    got, want = _both(ctx, reference, CSV_CASES[i], "csv")
    assert got == want


def test_raw_large_random(ctx, reference):
    rng = np.random.default_rng(5)
    L = rng.integers(1, 131073, size=300_000)
    pad = rng.choice([b"", b" ", b"\t", b"\r"], size=len(L))
    text = b"".join(p + str(int(v)).encode() + q + b"\n" for v, p, q in zip(L, pad, pad[::-1]))
    got = ctx.load_lengths(text, "raw-lengths")
    assert np.array_equal(got, L)
    assert np.array_equal(reference.load_lengths(text, "raw-lengths")[1], L)


def test_csv_device_output(ctx, reference):
    import torch
    rng = np.random.default_rng(6)
    L = rng.integers(1, 70000, size=100_000)
    text = b"id,length,source\n" + b"".join(b"%d,%d,web\n" % (i, v) for i, v in enumerate(L))
    out = torch.zeros(len(L), dtype=torch.int64, device="cuda")
    n = ctx.load_lengths(text, "csv", device_out=out)
    assert n == len(L) and np.array_equal(out.cpu().numpy(), L)
    assert np.array_equal(reference.load_lengths(text, "csv")[1], L)
