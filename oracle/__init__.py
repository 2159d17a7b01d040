"""TEST INFRASTRUCTURE ONLY: ctypes binding of the plain C oracle (oracle.c).

The oracle is a slow, obviously-correct CPU interpreter of the LTL4-C
semantics of arXiv:1411.2239 (see oracle.c's header for the passages each part
follows).  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It
shares no code with the product package ``paper_1411_2239_b200``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

VERDICT_NAMES = ["FALSE", "CURRENTLY_FALSE", "PRESUMABLY_FALSE",
                 "PRESUMABLY_TRUE", "CURRENTLY_TRUE", "TRUE"]
ABSENT = 0xFFFFFFFF
MAX_LEVELS = 3

ERRORS = {1: "syntax", 2: "noncanonical", 3: "unbound", 4: "range", 5: "budget"}


class OracleParseError(ValueError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code
        self.kind = ERRORS.get(code, str(code))


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C11, -O2)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-Wall", "-pthread",
                               "-Wno-format-truncation", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = ctypes.CDLL(build())
            c_u64p = ctypes.POINTER(ctypes.c_uint64)
            L.orc_parse.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p),
                                    ctypes.c_char_p, ctypes.c_int]
            L.orc_parse.restype = ctypes.c_int
            L.orc_prop_free.argtypes = [ctypes.c_void_p]
            L.orc_num_levels.argtypes = [ctypes.c_void_p]
            L.orc_num_atoms.argtypes = [ctypes.c_void_p]
            L.orc_atom_name.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_char_p, ctypes.c_int]
            L.orc_quantifier.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                         ctypes.POINTER(ctypes.c_int), c_u64p, c_u64p,
                                         ctypes.c_char_p, ctypes.c_int]
            L.orc_ltl4_word.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int]
            L.orc_fltl_word.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_int]
            L.orc_rule.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, c_u64p]
            L.orc_monitor_new.argtypes = [ctypes.c_void_p]
            L.orc_monitor_new.restype = ctypes.c_void_p
            L.orc_monitor_free.argtypes = [ctypes.c_void_p]
            L.orc_feed.argtypes = [ctypes.c_void_p, ctypes.c_uint64,
                                   ctypes.POINTER(ctypes.c_void_p), ctypes.c_void_p]
            L.orc_evaluate.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int), c_u64p,
                                       c_u64p, c_u64p]
            L.orc_node_verdict.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
            L.orc_run_threads.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.POINTER(ctypes.c_void_p),
                                          ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int), c_u64p,
                                          c_u64p, c_u64p]
            L.orc_reader_new.argtypes = [ctypes.c_void_p]
            L.orc_reader_new.restype = ctypes.c_void_p
            L.orc_reader_free.argtypes = [ctypes.c_void_p]
            L.orc_feed_jsonl.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_char_p, ctypes.c_uint64]
            L.orc_feed_jsonl.restype = ctypes.c_int64
            _lib = L
    return _lib


class Property:
    """A parsed LTL4-C property (Def. 3)."""

    def __init__(self, text: str):
        L = lib()
        h = ctypes.c_void_p()
        err = ctypes.create_string_buffer(256)
        rc = L.orc_parse(text.encode(), ctypes.byref(h), err, 256)
        if rc != 0:
            raise OracleParseError(rc, err.value.decode())
        self._h = h
        self.text = text

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_prop_free(self._h)
            self._h = None

    @property
    def levels(self) -> int:
        return lib().orc_num_levels(self._h)

    @property
    def atoms(self) -> list[str]:
        L = lib()
        out = []
        for j in range(L.orc_num_atoms(self._h)):
            b = ctypes.create_string_buffer(128)
            L.orc_atom_name(self._h, j, b, 128)
            out.append(b.value.decode())
        return out

    def quantifier(self, i: int) -> dict:
        L = lib()
        kind, cmp = ctypes.c_int(), ctypes.c_int()
        num, den = ctypes.c_uint64(), ctypes.c_uint64()
        key = ctypes.create_string_buffer(64)
        if L.orc_quantifier(self._h, i, ctypes.byref(kind), ctypes.byref(cmp), ctypes.byref(num),
                            ctypes.byref(den), key, 64) != 0:
            raise IndexError(i)
        return {"kind": "AE"[kind.value], "cmp": ["<", "<=", ">", ">=", "="][cmp.value],
                "num": num.value, "den": den.value, "key": key.value.decode()}

    def ltl4(self, word) -> int:
        """[u |=_4 psi] of the inner formula on one word (list of letters)."""
        w = bytes(bytearray(word))
        return lib().orc_ltl4_word(self._h, w, len(w))

    def fltl(self, word) -> int:
        w = bytes(bytearray(word))
        return lib().orc_fltl_word(self._h, w, len(w))


def rule(kind: str, cmp: str, num: int, den: int, h) -> int:
    """Def. 6 node verdict from a child-verdict histogram h[0..5]."""
    arr = (ctypes.c_uint64 * 6)(*[int(x) for x in h])
    return lib().orc_rule("AE".index(kind), ["<", "<=", ">", ">=", "="].index(cmp),
                          num, den, arr)


class Monitor:
    """Algorithm 1 run by the oracle: feed batches, evaluate the tree."""

    def __init__(self, prop: Property):
        self.prop = prop
        self._h = lib().orc_monitor_new(prop._h)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_monitor_free(self._h)
            self._h = None

    def feed(self, keys, letters):
        """keys: sequence of n uint32 arrays (one per level); letters: uint8 array."""
        n = self.prop.levels
        letters = np.ascontiguousarray(letters, dtype=np.uint8)
        ks = [np.ascontiguousarray(k, dtype=np.uint32) for k in keys]
        assert len(ks) >= n
        ptrs = (ctypes.c_void_p * MAX_LEVELS)()
        for i in range(n):
            assert ks[i].shape[0] == letters.shape[0]
            ptrs[i] = ks[i].ctypes.data
        lib().orc_feed(self._h, letters.shape[0], ptrs, letters.ctypes.data)

    def evaluate(self) -> dict:
        v = ctypes.c_int()
        hist = (ctypes.c_uint64 * ((MAX_LEVELS + 1) * 6))()
        seen, bound = ctypes.c_uint64(), ctypes.c_uint64()
        lib().orc_evaluate(self._h, ctypes.byref(v), hist, ctypes.byref(seen), ctypes.byref(bound))
        n = self.prop.levels
        h = np.array(list(hist), dtype=np.uint64).reshape(MAX_LEVELS + 1, 6)[: n + 1]
        return {"verdict": v.value, "hist": h, "events_seen": seen.value,
                "events_bound": bound.value}

    def node_verdict(self, prefix) -> int:
        arr = np.ascontiguousarray(prefix, dtype=np.uint32)
        return lib().orc_node_verdict(self._h, len(arr), arr.ctypes.data if len(arr) else None)


class RecordMonitor(Monitor):
    """A Monitor fed from JSON-lines records by the oracle's own reader."""

    def __init__(self, prop: Property):
        super().__init__(prop)
        self._r = lib().orc_reader_new(prop._h)

    def __del__(self):
        if getattr(self, "_r", None) and _lib is not None:
            _lib.orc_reader_free(self._r)
            self._r = None
        super().__del__()

    def feed_records(self, text) -> int:
        data = text.encode() if isinstance(text, str) else bytes(text)
        n = lib().orc_feed_jsonl(self._r, self._h, data, len(data))
        if n < 0:
            raise ValueError(f"malformed record on line {-n}")
        return n


def run_records(text: str, records) -> dict:
    """Algorithm 1 offline over JSON-lines records (the oracle's own reader)."""
    m = RecordMonitor(Property(text))
    m.feed_records(records)
    return m.evaluate()


def run_offline(text: str, keys, letters, threads: int = 1) -> dict:
    """Algorithm 1 offline.  threads > 1: the timing mode (orc_run_threads), level-0
    subtrees partitioned by a hash of k0 over `threads` host threads."""
    p = Property(text)
    if threads <= 1 or p.levels < 1:
        m = Monitor(p)
        m.feed(keys, letters)
        return m.evaluate()
    n = p.levels
    letters = np.ascontiguousarray(letters, dtype=np.uint8)
    ks = [np.ascontiguousarray(k, dtype=np.uint32) for k in keys[:n]]
    ptrs = (ctypes.c_void_p * MAX_LEVELS)()
    for i in range(n):
        ptrs[i] = ks[i].ctypes.data
    v = ctypes.c_int()
    hist = (ctypes.c_uint64 * ((MAX_LEVELS + 1) * 6))()
    seen, bound = ctypes.c_uint64(), ctypes.c_uint64()
    rc = lib().orc_run_threads(p._h, letters.shape[0], ptrs, letters.ctypes.data, int(threads),
                               ctypes.byref(v), hist, ctypes.byref(seen), ctypes.byref(bound))
    assert rc == 0
    h = np.array(list(hist), dtype=np.uint64).reshape(MAX_LEVELS + 1, 6)[: n + 1]
    return {"verdict": v.value, "hist": h, "events_seen": seen.value, "events_bound": bound.value}
