"""CPU tests of the host trace encoder (ltl4c_encode_jsonl; §4.1 Valuation
Extraction) against the oracle's own, independently written record
reader (oracle/oracle.c orc_feed_jsonl) and the paper's worked example written
as key -> value records (tests/golden/login_example.jsonl)."""
import os

import numpy as np
import pytest

import oracle
import paper_1411_2239_b200 as ltl4c
import tracegen

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
T, Tc, Tp, Fp, Fc, F = 5, 4, 3, 2, 1, 0


def test_worked_example_records_P715():
    """P:718-722 as records: 5 vectors, B(Adam, T) = 4 -> Adam F, root F
    (P:767), Jack Tc (reading A4) -- through the encoder and through the oracle's reader."""
    text = open(os.path.join(GOLDEN, "login_example.jsonl")).read()
    prog = ltl4c.compile(tracegen.LOGIN)
    keys, letters = prog.encoder().encode(text)
    assert [list(k) for k in keys] == [[0, 0, 1, 0, 0], [0, 1, 2, 3, 4]]
    assert list(letters) == [3, 3, 1, 3, 3]
    for r in (oracle.run_offline(tracegen.LOGIN, keys, letters), oracle.run_records(tracegen.LOGIN, text)):
        assert r["verdict"] == F
        assert list(r["hist"][2][[T, F]]) == [4, 1]
        assert list(r["hist"][1][[F, Tc]]) == [1, 1]


def _enc(formula, text):
    return ltl4c.compile(formula).encoder().encode(text)


def test_value_identity_is_canonical():
    """Numbers are identified by value (12 = 12.0 = 1.2e1 = "12"); strings as written."""
    f = "forall x : k(x) => F a"
    keys, _ = _enc(f, '{"k": 12}\n{"k": 12.0}\n{"k": 1.2e1}\n{"k": "12"}\n{"k": 120e-1}\n'
                      '{"k": "12.0"}\n{"k": -0}\n{"k": 0.0}\n{"k": "0"}\n{"k": "a\\u00e9"}\n{"k": "aé"}\n')
    assert list(keys[0]) == [0, 0, 0, 0, 0, 1, 2, 2, 2, 3, 3]


def test_non_scalar_values_bind_nothing():
    f = "forall x : k(x) => F a"
    keys, letters = _enc(f, '{"k": true}\n{"k": null}\n{"k": [1]}\n{"k": {"v": 1}}\n{"a": true}\n'
                            '{"k": 5, "a": false}\n{"k": 5, "a": 5}\n{"k": 5, "a": true, "k": 6}\n')
    A = 0xFFFFFFFF
    assert list(keys[0]) == [A, A, A, A, A, 0, 0, 1]
    assert list(letters) == [0, 0, 0, 0, 1, 0, 0, 1]   # a 0-ary atom holds only for `true`


def test_parametric_atoms_reading_A12():
    f = "forall x : k0(x) => forall y : k1(y) => F (p(x) && q(x, y) && r)"
    text = ('{"k0": 1, "k1": 2, "p": 1, "q": [1, 2], "r": true}\n'
            '{"k0": 1, "k1": 2, "p": 2, "q": [2, 1]}\n'
            '{"k0": 1, "k1": 2, "p": true, "q": true}\n'
            '{"k0": 1, "k1": 2, "p": "1", "q": [1.0, "2"]}\n'
            '{"k0": 1, "p": 1, "q": [1, 2]}\n')
    prog = ltl4c.compile(f)
    assert prog.atoms == ["p(x)", "q(x,y)", "r"]
    _, letters = prog.encoder().encode(text)
    assert list(letters) == [7, 0, 3, 3, 1]
    r = oracle.RecordMonitor(oracle.Property(f))
    r.feed_records(text)
    keys, _ = prog.encoder().encode(text)
    a, b = r.evaluate(), oracle.run_offline(f, keys, letters)
    assert a["verdict"] == b["verdict"] and np.array_equal(a["hist"], b["hist"])


def test_syntax_errors_and_resume():
    prog = ltl4c.compile(tracegen.LOGIN)
    enc = prog.encoder()
    for bad in ('{"user": 1,}', '[1, 2]', '{"user": tru}', '{"user": "x}', '{"user": 1} x', '{"user": 01x}'):
        with pytest.raises(ltl4c.Ltl4cError) as e:
            enc.encode(bad)
        assert e.value.name == "E_SYNTAX"
    # capacity-limited encoding resumes at the consumed byte offset
    import ctypes
    text = open(os.path.join(GOLDEN, "login_example.jsonl")).read().encode()
    lib = ltl4c._lib
    h = ctypes.c_void_p()
    assert lib.ltl4c_encoder_create(prog._h, ctypes.byref(h)) == 0
    keys = [np.zeros(2, np.uint32) for _ in range(2)]
    let = np.zeros(2, np.uint8)
    kp = (ctypes.c_void_p * 3)(keys[0].ctypes.data, keys[1].ctypes.data, None)
    n, used = ctypes.c_uint64(), ctypes.c_uint64()
    got_u, got_r, off = [], [], 0
    while off < len(text):
        assert lib.ltl4c_encode_jsonl(h, text[off:], len(text) - off, kp, let.ctypes.data, 2,
                                      ctypes.byref(n), ctypes.byref(used)) == 0
        got_u += list(keys[0][:n.value])
        got_r += list(keys[1][:n.value])
        off += used.value
    lib.ltl4c_encoder_free(h)
    assert got_u == [0, 0, 1, 0, 0] and got_r == [0, 1, 2, 3, 4]


CASES = {
    "C1": (lambda: tracegen.socket_trace(seed=3), ["socket"], ["receive", "respond"], [[0], [0]]),
    "C2": (lambda: tracegen.login_trace(seed=3, n=20_000, users=300, rid_events=2, p_unauth=0.1),
           ["user", "rid"], ["login", "unauthorized"], [[], []]),
    "C4": (lambda: tracegen.proxy_trace(seed=3, n=20_000, videos=500, p_ext_cached=0.02),
           ["vid", "req"], ["cached", "external"], [[0], [1]]),
}


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("style", ["plain", "mixed"])
def test_encoder_agrees_with_oracle_reader(name, style):
    """Workload-shaped record files: (product encoder -> oracle on the encoded arrays)
    = (oracle's own record reader) = (oracle on the generator's arrays)."""
    gen, keys_, preds, args = CASES[name]
    tr = gen()
    text = tracegen.to_jsonl(tr, keys_, preds, args, seed=1, style=style)
    k, l = ltl4c.compile(tr.formula).encoder().encode(text)
    a = oracle.run_offline(tr.formula, k, l)
    b = oracle.run_records(tr.formula, text)
    c = oracle.run_offline(tr.formula, tr.keys, tr.letters)
    for x in (b, c):
        assert a["verdict"] == x["verdict"] and np.array_equal(a["hist"], x["hist"]), name
        assert a["events_bound"] == x["events_bound"]
