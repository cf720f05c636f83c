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


JSONL_CASES = [
    b'{"length":4096}\n{"length":131072}\n', b'{"id":7,"length":10}\n\n{"length":20}\n',
    b'  {"length" : 5 , "x": [1, {"a": [true, false, null]}, "s"]}  \r\n{"length":6}',
    b'{"\\u006cength":9, "i\\u0064": -4}\n', b'{"length":1,"length":2}\n', b'{"id":"a","length":3}\n',
    b'{"id":3,"id":1.5,"length":3}\n', b'\xef\xbb\xbf{"length":8}\n', b'{"length":8, "k": "\xc3\xa9\xe2\x82\xac\xf0\x9f\x98\x80"}\n',
    b'{"s":"\\ud83d\\ude00 \\n\\t\\"\\\\\\/","length":11}\n', b'{"length":12,"n":-0.5e+3}\n',
    b'{"length":1}\n' * 4000, b'{"length":5,"id":18446744073709551615}\n',
    # errors
    b'', b'\n \n', b'{"length":0}\n', b'{"length":-3}\n', b'{"length":1.0}\n', b'{"length":"5"}\n', b'[1,2]\n',
    b'{"len":5}\n', b'{"length":5}x\n', b'{"length":5\n', b'{"length":05}\n', b'{"length":5,}\n',
    b'{"length":tru}\n', b'{"a":"\x01","length":1}\n', b'{"a":"\\x","length":1}\n', b'{"a":"\xff","length":1}\n',
    b'{"a":"\\ud800","length":1}\n', b'{"a":"\\udc00","length":1}\n', b'{"a":"\xed\xa0\x80","length":1}\n',
    b'{"length":18446744073709551615}\n', b'{"length":18446744073709551616}\n', b'{"length":-9223372036854775809}\n',
    b'{"id":1,"length":2}\n{"id":1,"length":3}\n', b'{"length":2}\n{"id":0,"length":3}\n',
    b'\xef\xbb{"length":8}\n', b'{"length":1}\n' * 3000 + b'{"length": 2,}\n', b'"x"\n', b'{} {}\n',
    b'{"length":2, "a":[' + b'[' * 50 + b']' * 50 + b']}\n', b'{"length":2, "a":[' + b'[' * 50 + b']' * 49 + b'}\n',
    b'{"length":5}\x00\n', b'{"length":5}\x00garbage\n', b'\x00{"length":5}\n', b'{"length":5\x00}\n', b'{"length":5,"v":1e}\n', b'{"length":5,"v":-}\n', b'{"length":5,"v":1.}\n',
]


def _both(ctx, oracle, text, fmt):
    try:
        want = ("ok",) + tuple(a.tolist() for a in oracle.load_lengths(text, fmt, "corpus.txt"))
    except Exception as e:  # noqa: BLE001
        want = (type(e).__name__, str(e))
    try:
        got = ("ok",) + tuple(a.tolist() for a in ctx.load_lengths(text, fmt, "corpus.txt", with_ids=True))
    except abi.ValidationError as e:
        got = ("ValidationError", str(e))
    return got, want


@pytest.mark.parametrize("i", range(len(JSONL_CASES)))
def test_jsonl(ctx, reference, i):
    got, want = _both(ctx, reference, JSONL_CASES[i], "jsonl")
    assert got == want


def test_jsonl_large_random(ctx, reference):
    rng = np.random.default_rng(8)
    L = rng.integers(1, 131073, size=200_000)
    ids = rng.permutation(10**6)[:len(L)] + 10**7  # explicit ids clear of the record indices
    rows = [(b'{"id":%d,"length":%d}' % (i, v)) if k % 3 else (b'{"length": %d, "src": "web"}' % v)
            for k, (i, v) in enumerate(zip(ids, L))]
    text = b"\n".join(rows) + b"\n"
    got_ids, got = ctx.load_lengths(text, "jsonl", with_ids=True)
    want_ids, want = reference.load_lengths(text, "jsonl")
    assert np.array_equal(got, L) and np.array_equal(got, want) and np.array_equal(got_ids, want_ids)


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


def test_jsonl_fuzz(ctx, reference):
    # single-line corpora from mutated records: the GPU's accept / reject
    # and the message must be the reference's (nlohmann) on every one
    rng = np.random.default_rng(11)
    base = [b'{"id":12,"length":345}', b'{"length": 7, "tags": ["a", {"b": null}], "f": -1.5e3}',
            b'{"\\u0069d": 3, "length": 9, "s": "x\\"y\\\\z\\u00e9"}', b'[{"length":1}]', b'{"length":true}']
    alphabet = list(b'{}[]:,"\\ -+.eE0123456789tfnulrsaxyz\t\r') + [0x00, 0x01, 0x7f, 0xc3, 0xa9, 0xff, 0xed, 0xf0]
    for k in range(1500):
        line = bytearray(base[k % len(base)])
        for _ in range(int(rng.integers(1, 4))):
            op = int(rng.integers(0, 3))
            pos = int(rng.integers(0, len(line) + 1))
            ch = int(alphabet[int(rng.integers(0, len(alphabet)))])
            if op == 0:
                line.insert(pos, ch)
            elif op == 1 and pos < len(line):
                del line[pos]
            elif pos < len(line):
                line[pos] = ch
        text = bytes(line).replace(b"\n", b" ") + b"\n"
        got, want = _both(ctx, reference, text, "jsonl")
        assert got == want, text


def test_golden_fixtures(ctx):
    # the committed outputs of the reference (tests/golden/make_ingest_golden.py)
    import json
    import os
    gold = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ingest_golden.json")))
    for g in gold:
        text = g["text"].encode("latin-1")
        try:
            ids, lens = ctx.load_lengths(text, g["format"], "corpus.txt", with_ids=True)
            got = {"ids": ids.tolist(), "lengths": lens.tolist()}
        except abi.ValidationError as e:
            got = {"error": str(e)}
        want = {k: g[k] for k in ("ids", "lengths", "error") if k in g}
        assert got == want, g["text"]
