"""paper_1411_2239_b200 -- B200-native LTL4-C runtime verification (arXiv:1411.2239).

Thin ctypes binding of ``libltl4c.so`` (C ABI in ``include/ltl4c.h``).  This
module only marshals arguments: compilation runs in the library's C++ compiler
and every step of the verification path runs in the library's sm_100a kernels.
There is no CPU fallback: if the library is missing this import fails, and a
state cannot be created without a B200.

    import paper_1411_2239_b200 as ltl4c
    prog = ltl4c.compile("forall x : user(x) => exists[<=3] r : rid(r) => (login && unauthorized)")
    st = prog.state(device=0)                 # offline; prog.state(online=True) for online mode
    res = st.verify([users, rids], letters)   # torch CUDA tensors (uint32 / int32 keys, uint8 letters)
    res[0].verdict, res[0].hist
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libltl4c.so")
if os.environ.get("LTL4C_LIB_VARIANT"):  # in-tree tuning variants (scripts/build_variant.sh)
    LIB_PATH = os.path.join(_HERE, f"libltl4c_{os.environ['LTL4C_LIB_VARIANT']}.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "ltl4c.h")

MAX_LEVELS = 3
MAX_FORMULAS = 4
MAX_KERNELS = 16
ABSENT = 0xFFFFFFFF
ONLINE = 1
VERDICTS = ["FALSE", "CURRENTLY_FALSE", "PRESUMABLY_FALSE", "PRESUMABLY_TRUE",
            "CURRENTLY_TRUE", "TRUE"]
STATUS = {0: "OK", 1: "E_SYNTAX", 2: "E_NONCANONICAL", 3: "E_UNBOUND", 4: "E_RANGE",
          5: "E_BUDGET", 6: "E_INVALID", 7: "E_CUDA", 8: "E_NCCL", 9: "E_OOM", 10: "E_POISONED"}

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(this package has no CPU fallback)")


class Ltl4cError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class _Quant(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("cmp", ctypes.c_int32), ("num", ctypes.c_uint64),
                ("den", ctypes.c_uint64), ("key", ctypes.c_char * 64)]


class _Tables(ctypes.Structure):
    _fields_ = [("n_formulas", ctypes.c_uint32), ("n_levels", ctypes.c_uint32),
                ("n_atoms", ctypes.c_uint32), ("n_states", ctypes.c_uint32),
                ("initial", ctypes.c_uint32), ("delta", ctypes.POINTER(ctypes.c_uint8)),
                ("label", ctypes.POINTER(ctypes.c_uint8)), ("quant", ctypes.POINTER(_Quant)),
                ("atom_names", ctypes.POINTER(ctypes.c_char_p)), ("letter_bits", ctypes.c_uint32),
                ("letter_class", ctypes.POINTER(ctypes.c_uint8))]


class _Batch(ctypes.Structure):
    _fields_ = [("n_events", ctypes.c_uint64), ("first_index", ctypes.c_uint64),
                ("keys", ctypes.c_void_p * MAX_LEVELS), ("letters", ctypes.c_void_p)]


class _Result(ctypes.Structure):
    _fields_ = [("verdict", ctypes.c_int32), ("n_levels", ctypes.c_uint32),
                ("hist", (ctypes.c_uint64 * 6) * (MAX_LEVELS + 1)),
                ("events_seen", ctypes.c_uint64), ("events_bound", ctypes.c_uint64)]


class _Stats(ctypes.Structure):
    _fields_ = [("verifies", ctypes.c_uint64), ("launches", ctypes.c_uint64),
                ("n_kernels", ctypes.c_uint32), ("kernel_name", (ctypes.c_char * 32) * MAX_KERNELS),
                ("kernel_launches", ctypes.c_uint64 * MAX_KERNELS),
                ("kernel_ms", ctypes.c_double * MAX_KERNELS)]


_lib = ctypes.CDLL(LIB_PATH)
_P = ctypes.c_void_p
_lib.ltl4c_compile.argtypes = [ctypes.c_char_p, ctypes.POINTER(_P)]
_lib.ltl4c_compile_batch.argtypes = [ctypes.POINTER(ctypes.c_char_p), ctypes.c_int, ctypes.POINTER(_P)]
_lib.ltl4c_program_tables.argtypes = [_P, ctypes.POINTER(_Tables)]
_lib.ltl4c_program_free.argtypes = [_P]
_lib.ltl4c_program_free.restype = None
_lib.ltl4c_state_create.argtypes = [_P, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint32, ctypes.POINTER(_P)]
_lib.ltl4c_state_comm.argtypes = [_P, ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
_lib.ltl4c_nccl_unique_id.argtypes = [ctypes.c_void_p]
_lib.ltl4c_nccl_unique_id.restype = ctypes.c_int
_lib.ltl4c_verify.argtypes = [_P, ctypes.POINTER(_Batch), ctypes.c_void_p, ctypes.POINTER(_Result)]
_lib.ltl4c_verify_host.argtypes = [_P, ctypes.POINTER(_Batch), ctypes.c_void_p, ctypes.POINTER(_Result)]
_lib.ltl4c_verify_async.argtypes = [_P, ctypes.POINTER(_Batch), ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64)]
_lib.ltl4c_result_get.argtypes = [_P, ctypes.c_uint64, ctypes.POINTER(_Result)]
_lib.ltl4c_state_reset.argtypes = [_P]
_lib.ltl4c_state_checkpoint_size.argtypes = [_P, ctypes.POINTER(ctypes.c_uint64)]
_lib.ltl4c_state_checkpoint.argtypes = [_P, ctypes.c_void_p, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64)]
_lib.ltl4c_state_restore.argtypes = [_P, ctypes.c_void_p, ctypes.c_uint64]
_lib.ltl4c_dencoder_create.argtypes = [_P, ctypes.c_int, ctypes.c_uint64, ctypes.POINTER(ctypes.c_void_p)]
_lib.ltl4c_dencode_jsonl.argtypes = [_P, ctypes.c_void_p, ctypes.c_uint64, ctypes.POINTER(ctypes.c_void_p),
                                     ctypes.c_void_p, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64), ctypes.c_void_p]
_lib.ltl4c_dencoder_values.argtypes = [_P, ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint64)]
_lib.ltl4c_dencoder_free.argtypes = [_P]
_lib.ltl4c_dencoder_free.restype = None
_lib.ltl4c_state_compact.argtypes = [_P]
_lib.ltl4c_state_nodes.argtypes = [_P, ctypes.c_uint32, ctypes.c_uint32, ctypes.POINTER(ctypes.c_void_p),
                                   ctypes.c_void_p, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64)]
_lib.ltl4c_state_free.argtypes = [_P]
_lib.ltl4c_state_free.restype = None
_lib.ltl4c_state_profile.argtypes = [_P, ctypes.c_int]
_lib.ltl4c_state_stats.argtypes = [_P, ctypes.POINTER(_Stats)]
_lib.ltl4c_state_stats_reset.argtypes = [_P]
_lib.ltl4c_encoder_create.argtypes = [_P, ctypes.POINTER(_P)]
_lib.ltl4c_encode_jsonl.argtypes = [_P, ctypes.c_char_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)]
_lib.ltl4c_encoder_values.argtypes = [_P, ctypes.c_uint32, ctypes.POINTER(ctypes.c_uint64)]
_lib.ltl4c_encoder_free.argtypes = [_P]
_lib.ltl4c_encoder_free.restype = None
_lib.ltl4c_last_error.restype = ctypes.c_char_p
_lib.ltl4c_version.restype = ctypes.c_char_p
for _fn in ("ltl4c_compile", "ltl4c_compile_batch", "ltl4c_program_tables", "ltl4c_state_create",
            "ltl4c_state_comm", "ltl4c_verify", "ltl4c_verify_host", "ltl4c_verify_async", "ltl4c_result_get",
            "ltl4c_state_reset",
            "ltl4c_state_profile", "ltl4c_state_stats", "ltl4c_state_stats_reset",
            "ltl4c_encoder_create", "ltl4c_encode_jsonl", "ltl4c_encoder_values"):
    getattr(_lib, _fn).restype = ctypes.c_int


def _check(st: int):
    if st != 0:
        raise Ltl4cError(st, _lib.ltl4c_last_error().decode(errors="replace"))


def version() -> str:
    return _lib.ltl4c_version().decode()


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId for ltl4c_state_comm (call on rank 0, broadcast)."""
    buf = ctypes.create_string_buffer(128)
    _check(_lib.ltl4c_nccl_unique_id(buf))
    return buf.raw


@dataclass
class Result:
    verdict: int
    hist: np.ndarray          # [n_levels + 1, 6]: depth 0 (root) .. n (leaves)
    events_seen: int
    events_bound: int

    @property
    def verdict_name(self) -> str:
        return VERDICTS[self.verdict]


class Program:
    """A compiled LTL4-C program: LTL4 monitor + quantifier string (immutable)."""

    def __init__(self, handle: ctypes.c_void_p, texts):
        self._h = handle
        self.texts = list(texts)
        t = _Tables()
        _check(_lib.ltl4c_program_tables(self._h, ctypes.byref(t)))
        self.n_formulas = t.n_formulas
        self.n_levels = t.n_levels
        self.n_atoms = t.n_atoms
        self.n_states = t.n_states
        self.initial = t.initial
        self.letter_bits = t.letter_bits
        A = 1 << t.letter_bits
        self.delta = np.ctypeslib.as_array(t.delta, shape=(t.n_states * A,)).reshape(t.n_states, A).copy()
        # letter code of each atom valuation (formula batches over > 8 atoms), or None
        self.letter_class = (np.ctypeslib.as_array(t.letter_class, shape=(1 << t.n_atoms,)).copy()
                             if bool(t.letter_class) else None)
        self.label = np.ctypeslib.as_array(t.label, shape=(t.n_formulas * t.n_states,)).reshape(
            t.n_formulas, t.n_states).copy()
        self.atoms = [t.atom_names[j].decode() for j in range(t.n_atoms)]
        self.quantifiers = []
        for f in range(t.n_formulas):
            row = []
            for l in range(t.n_levels):
                q = t.quant[f * t.n_levels + l]
                row.append({"kind": "AE"[q.kind], "cmp": ["<", "<=", ">", ">=", "="][q.cmp],
                            "num": q.num, "den": q.den, "key": q.key.decode()})
            self.quantifiers.append(row)

    def __del__(self):
        try:
            if getattr(self, "_h", None) and _lib is not None:
                _lib.ltl4c_program_free(self._h)
        except Exception:
            pass
        self._h = None

    def state(self, device: int = 0, online: bool = False, capacity: int = 0) -> "State":
        return State(self, device, online, capacity)

    def codes(self, valuations) -> np.ndarray:
        """Letter codes of atom valuations (bit j = atom j): the valuations themselves up
        to 8 atoms, their letter classes beyond (ltl4c_tables.letter_class)."""
        v = np.asarray(valuations)
        if self.letter_class is None:
            return v.astype(np.uint8)
        return self.letter_class[v.astype(np.int64)]

    def encoder(self) -> "Encoder":
        """Host trace encoder for this program's guard keys and atoms (ltl4c_encode_jsonl)."""
        return Encoder(self)

    def device_encoder(self, device: int = 0, max_values: int = 1 << 22) -> "DeviceEncoder":
        """Trace encoder on the GPU (ltl4c_dencode_jsonl)."""
        return DeviceEncoder(self, device, max_values)


class Encoder:
    """JSON-lines records -> (keys, letters) host arrays in the layout verify() takes
    (ltl4c_encode_jsonl: per-key dictionaries persist across calls)."""

    def __init__(self, prog: Program):
        self.prog = prog
        self._h = ctypes.c_void_p()
        _check(_lib.ltl4c_encoder_create(prog._h, ctypes.byref(self._h)))

    def __del__(self):
        try:
            if getattr(self, "_h", None) and _lib is not None:
                _lib.ltl4c_encoder_free(self._h)
        except Exception:
            pass
        self._h = None

    def encode(self, text) -> tuple[list[np.ndarray], np.ndarray]:
        """Encode every record of `text` (str or bytes, one JSON object per line)."""
        data = text.encode() if isinstance(text, str) else bytes(text)
        cap = data.count(b"\n") + 1
        keys = [np.empty(cap, np.uint32) for _ in range(self.prog.n_levels)]
        letters = np.empty(cap, np.uint8)
        kp = (ctypes.c_void_p * MAX_LEVELS)(*[k.ctypes.data for k in keys])
        n, used = ctypes.c_uint64(), ctypes.c_uint64()
        _check(_lib.ltl4c_encode_jsonl(self._h, data, len(data), kp, letters.ctypes.data, cap,
                                       ctypes.byref(n), ctypes.byref(used)))
        m = int(n.value)
        return [k[:m].copy() for k in keys], letters[:m].copy()

    def values(self, level: int) -> int:
        c = ctypes.c_uint64()
        _check(_lib.ltl4c_encoder_values(self._h, level, ctypes.byref(c)))
        return int(c.value)


class DeviceEncoder:
    """JSON-lines records already in device memory -> (keys, letters) device tensors
    (ltl4c_dencode_jsonl: the host encoder's semantics on the GPU; per-key
    dictionaries persist across calls; ids are a relabelling of the host encoder's)."""

    def __init__(self, prog: Program, device: int, max_values: int):
        self.prog, self.device = prog, device
        self._h = ctypes.c_void_p()
        _check(_lib.ltl4c_dencoder_create(prog._h, device, max_values, ctypes.byref(self._h)))

    def __del__(self):
        try:
            if getattr(self, "_h", None) and _lib is not None:
                _lib.ltl4c_dencoder_free(self._h)
        except Exception:
            pass
        self._h = None

    def encode(self, text, stream=None):
        """`text`: a uint8 CUDA tensor of JSON lines (or bytes / str, copied to the
        device first).  Returns (keys: list of int32 device tensors, letters: uint8
        device tensor), one event per record."""
        import torch
        dev = torch.device("cuda", self.device)
        if not isinstance(text, torch.Tensor):
            data = text.encode() if isinstance(text, str) else bytes(text)
            text = torch.frombuffer(bytearray(data), dtype=torch.uint8).to(dev) if data else torch.zeros(0, dtype=torch.uint8, device=dev)
        n_nl = int((text == 10).sum().item()) if text.numel() else 0
        cap = n_nl + 1
        keys = [torch.empty(cap, dtype=torch.int32, device=dev) for _ in range(self.prog.n_levels)]
        letters = torch.empty(cap, dtype=torch.uint8, device=dev)
        kp = (ctypes.c_void_p * MAX_LEVELS)(*[k.data_ptr() for k in keys])
        n = ctypes.c_uint64()
        _check(_lib.ltl4c_dencode_jsonl(self._h, ctypes.c_void_p(text.data_ptr() if text.numel() else 0),
                                        text.numel(), kp, ctypes.c_void_p(letters.data_ptr()), cap,
                                        ctypes.byref(n), _stream_handle(stream)))
        m = int(n.value)
        return [k[:m] for k in keys], letters[:m]

    def encode_into(self, text, keys, letters, stream=None) -> int:
        """As encode(), into caller-allocated device buffers (int32 key tensors, a uint8
        letter tensor; capacity = letters.numel()): no host-side pass over the text and
        no allocation.  Returns the number of events written."""
        kp = (ctypes.c_void_p * MAX_LEVELS)(*[k.data_ptr() for k in keys])
        n = ctypes.c_uint64()
        _check(_lib.ltl4c_dencode_jsonl(self._h, ctypes.c_void_p(text.data_ptr() if text.numel() else 0),
                                        text.numel(), kp, ctypes.c_void_p(letters.data_ptr()), letters.numel(),
                                        ctypes.byref(n), _stream_handle(stream)))
        return int(n.value)

    def values(self, level: int) -> int:
        c = ctypes.c_uint64()
        _check(_lib.ltl4c_dencoder_values(self._h, level, ctypes.byref(c)))
        return int(c.value)


def compile(text: str) -> Program:  # noqa: A001 (mirrors ltl4c_compile)
    h = ctypes.c_void_p()
    _check(_lib.ltl4c_compile(text.encode(), ctypes.byref(h)))
    return Program(h, [text])


def compile_batch(texts) -> Program:
    arr = (ctypes.c_char_p * len(texts))(*[t.encode() for t in texts])
    h = ctypes.c_void_p()
    _check(_lib.ltl4c_compile_batch(arr, len(texts), ctypes.byref(h)))
    return Program(h, texts)


def _stream_handle(stream):
    if stream is None:
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if hasattr(stream, "cuda_stream"):
        return ctypes.c_void_p(stream.cuda_stream)
    return ctypes.c_void_p(int(stream))


class State:
    """Verification state on one B200 (carried submonitor tree when online)."""

    def __init__(self, prog: Program, device: int, online: bool, capacity: int):
        self.prog = prog
        self.device = device
        self.online = online
        self._h = ctypes.c_void_p()
        _check(_lib.ltl4c_state_create(prog._h, device, capacity, ONLINE if online else 0,
                                       ctypes.byref(self._h)))
        self.next_index = 0
        self._pending = {}  # ticket -> input tensors of a pipelined batch

    def __del__(self):
        try:
            if getattr(self, "_h", None) and _lib is not None:
                _lib.ltl4c_state_free(self._h)
        except Exception:
            pass
        self._h = None

    def _results(self, res) -> list[Result]:
        n = self.prog.n_levels
        out = []
        for f in range(self.prog.n_formulas):
            r = res[f]
            h = np.array([[r.hist[l][v] for v in range(6)] for l in range(n + 1)], dtype=np.uint64)
            out.append(Result(int(r.verdict), h, int(r.events_seen), int(r.events_bound)))
        return out

    def _batch(self, keys, letters, n, first_index, ptr):
        b = _Batch()
        b.n_events = n
        b.first_index = self.next_index if first_index is None else first_index
        for i in range(self.prog.n_levels):
            b.keys[i] = ptr(keys[i])
        b.letters = ptr(letters)
        return b

    def verify(self, keys, letters, first_index=None, stream=None) -> list[Result]:
        """keys: n_levels CUDA tensors (uint32 or int32 bit patterns), letters: uint8 CUDA tensor."""
        import torch
        n = int(letters.numel())
        for k in list(keys)[: self.prog.n_levels]:
            if not (k.is_cuda and k.is_contiguous() and k.element_size() == 4 and k.numel() == n):
                raise ValueError("keys must be contiguous 4-byte CUDA tensors of the same length as letters")
        if not (letters.is_cuda and letters.is_contiguous() and letters.dtype == torch.uint8):
            raise ValueError("letters must be a contiguous uint8 CUDA tensor")
        b = self._batch(keys, letters, n, first_index, lambda t: t.data_ptr() if n else None)
        res = (_Result * self.prog.n_formulas)()
        _check(_lib.ltl4c_verify(self._h, ctypes.byref(b), _stream_handle(stream), res))
        self.next_index = b.first_index + n
        return self._results(res)

    def verify_async(self, keys, letters, first_index=None, stream=None) -> int:
        """Online states: enqueue one batch and return a ticket at once (the result is
        read with result(ticket); the tensors are kept alive until then)."""
        import torch
        n = int(letters.numel())
        keys = list(keys)[: self.prog.n_levels]
        for k in keys:
            if not (k.is_cuda and k.is_contiguous() and k.element_size() == 4 and k.numel() == n):
                raise ValueError("keys must be contiguous 4-byte CUDA tensors of the same length as letters")
        if not (letters.is_cuda and letters.is_contiguous() and letters.dtype == torch.uint8):
            raise ValueError("letters must be a contiguous uint8 CUDA tensor")
        b = self._batch(keys, letters, n, first_index, lambda t: t.data_ptr() if n else None)
        t = ctypes.c_uint64()
        _check(_lib.ltl4c_verify_async(self._h, ctypes.byref(b), _stream_handle(stream), ctypes.byref(t)))
        self.next_index = b.first_index + n
        self._pending[t.value] = (keys, letters)
        return t.value

    def result(self, ticket: int) -> list[Result]:
        """Wait for the batch of `ticket` (from verify_async) and return its result."""
        res = (_Result * self.prog.n_formulas)()
        try:
            _check(_lib.ltl4c_result_get(self._h, ticket, res))
        finally:
            self._pending.pop(ticket, None)
        return self._results(res)

    def verify_host(self, keys, letters, first_index=None, stream=None) -> list[Result]:
        """As verify(), with host arrays (numpy or pinned torch CPU tensors); the
        host->device copies run inside the library call."""
        def ptr(a):
            if hasattr(a, "data_ptr"):
                return a.data_ptr()
            return a.ctypes.data
        n = int(letters.shape[0])
        keep = [np.ascontiguousarray(k, dtype=np.uint32) if isinstance(k, np.ndarray) else k
                for k in list(keys)[: self.prog.n_levels]]
        let = np.ascontiguousarray(letters, dtype=np.uint8) if isinstance(letters, np.ndarray) else letters
        b = self._batch(keep, let, n, first_index, lambda a: ptr(a) if n else None)
        res = (_Result * self.prog.n_formulas)()
        _check(_lib.ltl4c_verify_host(self._h, ctypes.byref(b), _stream_handle(stream), res))
        self.next_index = b.first_index + n
        return self._results(res)

    def comm(self, nccl_id: bytes, n_ranks: int, rank: int):
        """Join an NCCL communicator (multi-GPU sharded verification)."""
        buf = ctypes.create_string_buffer(bytes(nccl_id), 128) if nccl_id is not None else None
        _check(_lib.ltl4c_state_comm(self._h, buf, n_ranks, rank))

    def reset(self):
        _check(_lib.ltl4c_state_reset(self._h))
        self.next_index = 0

    def checkpoint(self) -> bytes:
        """The carried state of an online state as an opaque blob (ltl4c_state_checkpoint)."""
        n = ctypes.c_uint64()
        _check(_lib.ltl4c_state_checkpoint_size(self._h, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(max(1, n.value))
        w = ctypes.c_uint64()
        _check(_lib.ltl4c_state_checkpoint(self._h, buf, n.value, ctypes.byref(w)))
        return bytes(buf.raw[:w.value]) + self.next_index.to_bytes(8, "little")

    def compact(self):
        """Shrink an online state's carried tables to its live entries (ltl4c_state_compact)."""
        _check(_lib.ltl4c_state_compact(self._h))

    def nodes(self, level: int, formula: int = 0):
        """(keys, verdicts) of every node at depth `level` of an online state's tree
        (level = n_levels: the leaves) -- ltl4c_state_nodes.  keys: list of `level`
        uint32 arrays; verdicts: uint8 B6 codes."""
        cnt = ctypes.c_uint64()
        _check(_lib.ltl4c_state_nodes(self._h, level, formula, None, None, 0, ctypes.byref(cnt)))
        n = cnt.value
        keys = [np.zeros(n, np.uint32) for _ in range(level)]
        ver = np.zeros(n, np.uint8)
        if n:
            ptrs = (ctypes.c_void_p * level)(*[k.ctypes.data for k in keys])
            _check(_lib.ltl4c_state_nodes(self._h, level, formula, ptrs, ver.ctypes.data, n, ctypes.byref(cnt)))
        return keys, ver

    def restore(self, blob: bytes):
        """Continue the stream of a checkpointed online state (ltl4c_state_restore)."""
        body, nxt = blob[:-8], int.from_bytes(blob[-8:], "little")
        buf = ctypes.create_string_buffer(body, len(body))
        _check(_lib.ltl4c_state_restore(self._h, buf, len(body)))
        self.next_index = nxt

    def profile(self, enable: bool = True):
        _check(_lib.ltl4c_state_profile(self._h, 1 if enable else 0))

    def stats(self) -> dict:
        s = _Stats()
        _check(_lib.ltl4c_state_stats(self._h, ctypes.byref(s)))
        kernels = {}
        for k in range(s.n_kernels):
            kernels[s.kernel_name[k].value.decode()] = {"launches": int(s.kernel_launches[k]),
                                                        "ms": float(s.kernel_ms[k])}
        return {"verifies": int(s.verifies), "launches": int(s.launches), "kernels": kernels}

    def stats_reset(self):
        _check(_lib.ltl4c_state_stats_reset(self._h))
