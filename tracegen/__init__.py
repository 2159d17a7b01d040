"""Seeded synthetic trace generators (shared by tests, bench and smoke).

This module holds NONE of the method's arithmetic: it only draws events.  Both
the oracle and the product path read the bytes it produces.  Each generator
returns a ``Trace`` with

* ``formula``  -- the LTL4-C property text the workload is shaped for,
* ``keys``     -- list of ``n_levels`` uint32 arrays (value of guard key i per
                  event; ``ABSENT`` = 0xFFFFFFFF when the event does not bind it),
* ``letters``  -- uint8 array; bit j = atom j of the formula, atoms numbered by
                  first occurrence in the formula's body.

Workload recipes follow SURVEY.md §8(d) / DESIGN.md "Input recipe":
C1 socket, C2 nested login (Eq. 8), C3 Zipf-skewed
socket, C4 proxy cache, C5 three-level online batch, C6 the
Dropbox fairness case study.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

ABSENT = np.uint32(0xFFFFFFFF)
SEED_BASE = 0x14112239

SOCKET = "forall[>=0.95] s : socket(s) => G (receive(s) -> F respond(s))"
LOGIN = "forall x : user(x) => exists[<=3] r : rid(r) => (login && unauthorized)"
PROXY = "forall v : vid(v) => exists[=0] r : req(r) => (cached(v) && external(r))"
FILES = "forall[>=50%] f : intrace(f) => (opened(f) U close(f))"
DROPBOX = "forall u : user(u) => F small(u)"
FIG1 = "forall[>=0.5] f : file(f) => (G a || (b U c))"
C5_FORMULAS = [
    "forall[>=0.95] h : host(h) => forall u : user(u) => exists[<=2] s : session(s) => F authfail",
    "exists[>=3] h : host(h) => forall[>=0.5] u : user(u) => forall s : session(s) => G (request -> F response)",
    "forall[>=0.99] h : host(h) => exists[=0] u : user(u) => exists s : session(s) => (admin && external)",
]


@dataclass
class Trace:
    formula: str
    keys: list
    letters: np.ndarray
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.letters.shape[0])


def _ids(rng: np.random.Generator, count: int) -> np.ndarray:
    """`count` distinct uint32 ids != ABSENT (a random odd-multiplier bijection)."""
    mul = np.uint64(rng.integers(1, 2**31) * 2 + 1)
    add = np.uint64(rng.integers(0, 2**32))
    i = np.arange(count, dtype=np.uint64)
    v = ((i * mul + add) & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    v[v == ABSENT] = np.uint32(0xFFFFFFFE)  # keep distinct in practice; collision prob ~0
    return v


def socket_trace(seed: int = 0, n: int = 10_000, sockets: int = 100, noise: float = 0.02,
                 p_receive: float = 0.04, p_respond: float = 0.95, p_drop: float = 0.005) -> Trace:
    """C1: web-server socket trace. bit0 = receive(s), bit1 = respond(s).

    Per event: with prob `noise` the event binds no socket; otherwise a socket is
    drawn uniformly from `sockets` fds in [0, 65535].  An idle socket
    receives a request with prob `p_receive`; a pending one is responded with prob
    `p_respond` unless the request was dropped (prob `p_drop`, never responded).
    """
    rng = np.random.default_rng(SEED_BASE + 1 + seed)
    fds = rng.choice(65536, size=sockets, replace=False).astype(np.uint32)
    sock = rng.integers(0, sockets, size=n)
    is_noise = rng.random(n) < noise
    u1, u2 = rng.random(n), rng.random(n)
    pending = np.zeros(sockets, dtype=np.int8)  # 0 idle, 1 pending, 2 dropped
    letters = np.zeros(n, dtype=np.uint8)
    keys = np.empty(n, dtype=np.uint32)
    for j in range(n):  # sequential per-socket state machine (small n only)
        if is_noise[j]:
            keys[j] = ABSENT
            continue
        s = sock[j]
        keys[j] = fds[s]
        if pending[s] == 0:
            if u1[j] < p_receive:
                letters[j] = 1
                pending[s] = 2 if u2[j] < p_drop else 1
        elif pending[s] == 1 and u1[j] < p_respond:
            letters[j] = 2
            pending[s] = 0
    return Trace(SOCKET, [keys], letters, {"config": "C1", "seed": seed, "sockets": sockets})


def login_trace(seed: int = 0, n: int = 10_000_000, users: int = 100_000, p_login: float = 0.3,
                p_unauth: float = 0.02, p_norid: float = 0.01, rid_events: int = 1,
                variant: str = "random") -> Trace:
    """C2: nested login property (Eq. 8).  bit0 = login, bit1 = unauthorized.

    Users uniform over `users` ids; request ids unique per request, each request
    spanning `rid_events` consecutive-in-request events (1 = unique per event);
    `p_norid` of events bind no rid.  variant: "random" | "clean" (every user
    has <= 3 login&unauthorized requests) | "violator" (clean + one user with 4).
    """
    rng = np.random.default_rng(SEED_BASE + 2 + seed)
    uid = _ids(rng, users)
    u = rng.integers(0, users, size=n)
    nreq = (n + rid_events - 1) // rid_events
    rids = _ids(rng, nreq)
    if rid_events == 1:
        r = rids
    else:
        # events of a request are spread over the trace: request k's events
        # take random positions (still one user per request)
        req_of = np.repeat(np.arange(nreq), rid_events)[:n]
        rng.shuffle(req_of)
        r = rids[req_of]
        req_user = rng.integers(0, users, size=nreq)
        u = req_user[req_of]
    login = rng.random(n) < p_login
    unauth = login & (rng.random(n) < p_unauth)
    letters = (login.astype(np.uint8) | (unauth.astype(np.uint8) << 1))
    rk = r.copy()
    rk[rng.random(n) < p_norid] = ABSENT
    uk = uid[u].astype(np.uint32)
    if variant in ("clean", "violator"):
        both = (letters == 3) & (rk != ABSENT)
        idx = np.nonzero(both)[0]
        order = np.argsort(u[idx], kind="stable")
        su = u[idx][order]
        start = np.r_[0, np.nonzero(np.diff(su))[0] + 1]
        rank = np.arange(su.shape[0]) - np.repeat(start, np.diff(np.r_[start, su.shape[0]]))
        drop = idx[order][rank >= 3]
        letters[drop] = 1  # keep login, clear unauthorized
        if variant == "violator":
            victim = int(u[0])
            pos = np.nonzero((u == victim) & (rk != ABSENT) & (letters != 3))[0][:4]
            letters[pos] = 3
            if rid_events != 1:
                pass
    return Trace(LOGIN, [uk, rk], letters,
                 {"config": "C2", "seed": seed, "users": users, "variant": variant})


BLOCK = 1 << 20  # events per independently generated block (C3, C4): any slice [lo, hi)
                 # of a trace can be generated alone (multi-GPU ranks generate their own)


def _blocks(n: int, lo: int, hi, fn):
    """Run fn(b, a, z) for every block b intersecting [lo, hi) (a, z = the part of
    block b inside the slice, block-relative), in parallel threads; returns the
    results in block order."""
    from concurrent.futures import ThreadPoolExecutor
    hi = n if hi is None else hi
    assert 0 <= lo <= hi <= n
    jobs = []
    for b in range(lo // BLOCK, (hi + BLOCK - 1) // BLOCK):
        a0, z0 = max(lo, b * BLOCK) - b * BLOCK, min(hi, (b + 1) * BLOCK) - b * BLOCK
        jobs.append((b, a0, z0))
    if len(jobs) <= 1:
        return [fn(*j) for j in jobs]
    import os
    with ThreadPoolExecutor(max_workers=min(len(jobs), max(1, (os.cpu_count() or 1)))) as ex:
        return list(ex.map(lambda j: fn(*j), jobs))


def _zipf_cdf(support: int, s: float) -> np.ndarray:
    w = np.arange(1, support + 1, dtype=np.float64) ** (-s)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    return cdf


def zipf_socket_trace(seed: int = 0, n: int = 100_000_000, support: int = 1 << 20, s: float = 1.1,
                      p_receive: float = 0.3, p_respond: float = 0.3, formula: str = SOCKET,
                      lo: int = 0, hi=None) -> Trace:
    """C3: Zipf(s)-skewed keys over `support` ids; i.i.d. letters over {receive, respond}
    (the G(r -> F s) automaton has two non-trap states, so every event does work).
    Events [lo, hi) of the n-event trace; blocks of BLOCK events are drawn from their
    own seeded stream, so any slice is generated alone."""
    ids = _ids(np.random.default_rng(SEED_BASE + 3 + seed), support)
    cdf = _zipf_cdf(support, s)
    blen = n  # events of the last block may be fewer

    def block(b, a0, z0):
        rng = np.random.default_rng([SEED_BASE + 3, seed, b])
        m = min(BLOCK, blen - b * BLOCK)
        r = np.searchsorted(cdf, rng.random(m), side="right")
        np.minimum(r, support - 1, out=r)
        let = ((rng.random(m) < p_receive).astype(np.uint8)
               | ((rng.random(m) < p_respond).astype(np.uint8) << 1))
        return ids[r[a0:z0]], let[a0:z0]

    parts = _blocks(n, lo, hi, block)
    keys = np.concatenate([p[0] for p in parts]) if parts else np.zeros(0, np.uint32)
    letters = np.concatenate([p[1] for p in parts]) if parts else np.zeros(0, np.uint8)
    return Trace(formula, [keys], letters, {"config": "C3", "seed": seed, "support": support, "s": s,
                                            "n": n, "lo": lo})


def _unique_id(i: np.ndarray, mul: int) -> np.ndarray:
    """bijection of [0, 2^32 - 1) onto u32 values != ABSENT: (i + 1) * mul - 1 mod 2^32"""
    return (((i.astype(np.uint64) + np.uint64(1)) * np.uint64(mul) - np.uint64(1))
            & np.uint64(0xFFFFFFFF)).astype(np.uint32)


def proxy_trace(seed: int = 0, n: int = 1_000_000, videos: int = 1_000_000, s: float = 0.8,
                p_cached: float = 0.6, p_ext: float = 0.5, p_ext_cached: float = 0.001,
                max_req_events: int = 4, lo: int = 0, hi=None) -> Trace:
    """C4: YouTube proxy cache. bit0 = cached(v), bit1 = external(r).
    Videos Zipf(s); requests unique with 1..max_req_events events each, each request's
    events placed near each other.  Events [lo, hi) of the n-event trace: every block
    of BLOCK events holds whole requests and is drawn from its own seeded stream (a
    request's id is unique over the whole trace), so any slice is generated alone."""
    grng = np.random.default_rng(SEED_BASE + 4 + seed)
    vids = _ids(grng, videos)
    rmul = int(grng.integers(1, 2**31)) * 2 + 1
    cdf = _zipf_cdf(videos, s)

    def block(b, a0, z0):
        rng = np.random.default_rng([SEED_BASE + 4, seed, b])
        m = min(BLOCK, n - b * BLOCK)
        per = rng.integers(1, max_req_events + 1, size=m // 2 + 1)
        cs = np.cumsum(per)
        nreq = int(np.searchsorted(cs, m) + 1)
        req_of = np.repeat(np.arange(nreq), per[:nreq])[:m]
        jitter = rng.random(m) * 64.0
        order = np.argsort(req_of.astype(np.float64) * 2.5 + jitter, kind="stable")
        req_of = req_of[order]
        vr = np.searchsorted(cdf, rng.random(nreq), side="right")
        np.minimum(vr, videos - 1, out=vr)
        rid = _unique_id(np.uint64(b) * np.uint64(BLOCK) + np.arange(nreq, dtype=np.uint64), rmul)
        cached_req = rng.random(nreq) < p_cached
        cached = cached_req[req_of]
        ext = np.where(cached, rng.random(m) < p_ext_cached, rng.random(m) < p_ext)
        let = cached.astype(np.uint8) | (ext.astype(np.uint8) << 1)
        sl = slice(a0, z0)
        return vids[vr[req_of[sl]]], rid[req_of[sl]], let[sl]

    parts = _blocks(n, lo, hi, block)
    cat = (lambda i, dt: np.concatenate([p[i] for p in parts]) if parts else np.zeros(0, dt))
    return Trace(PROXY, [cat(0, np.uint32), cat(1, np.uint32)], cat(2, np.uint8),
                 {"config": "C4", "seed": seed, "videos": videos, "n": n, "lo": lo})


def dropbox_trace(seed: int = 0, n: int = 1_000_000, users: int = 10_000, chunk_max: float = 4.0,
                  p_heavy: float = 0.02) -> Trace:
    """C6: personal cloud storage fairness: A u : user(u) => F small(u),
    small(u) = avg_chunksize(u) <= maximum.  Each event is one chunk upload by a user
    (uniform over `users`); a user's chunk sizes are exponential with a per-user mean
    (most users well below `chunk_max`; a fraction `p_heavy` repeatedly upload chunks of
    about the maximum size); bit0 of the letter = the user's running average
    chunk size over their uploads so far is <= chunk_max (the program variable the
    predicate reads).  No method arithmetic: the atom is part of the input."""
    rng = np.random.default_rng(SEED_BASE + 6 + seed)
    ids = _ids(rng, users)
    heavy = rng.random(users) < p_heavy
    mean = np.where(heavy, chunk_max * 1.02, rng.uniform(0.2, 1.5, users) * chunk_max)
    u = rng.integers(0, users, n)
    size = rng.exponential(1.0, n) * mean[u]
    size = np.where(heavy[u], chunk_max * (1.0 + 0.05 * rng.random(n)), size)
    order = np.argsort(u, kind="stable")            # per-user running averages in trace order
    su, ss = u[order], size[order]
    csum = np.cumsum(ss)
    first = np.r_[True, su[1:] != su[:-1]]
    start = np.maximum.accumulate(np.where(first, np.arange(n), 0))
    base = np.where(start > 0, csum[start - 1], 0.0)
    cnt = np.arange(n) - start + 1
    avg = (csum - base) / cnt
    small = np.empty(n, dtype=np.uint8)
    small[order] = (avg <= chunk_max).astype(np.uint8)
    return Trace(DROPBOX, [ids[u]], small, {"config": "C6", "seed": seed, "users": users, "n": n})


def worked_example() -> Trace:
    """The five-event login trace of P:715-723 (Adam = 1, Jack = 2)."""
    users = np.array([1, 1, 2, 1, 1], dtype=np.uint32)
    rids = np.array([12, 13, 14, 15, 16], dtype=np.uint32)
    letters = np.array([3, 3, 1, 3, 3], dtype=np.uint8)  # Jack: login, authorized
    return Trace(LOGIN, [users, rids], letters, {"config": "worked-example"})


def random_property_trace(seed: int, levels: int, n_events: int, values: int = 3,
                          atoms: int = 2, p_absent: float = 0.1):
    """Small random trace for property-based tests (keys in [0, values))."""
    rng = np.random.default_rng(SEED_BASE + 100 + seed)
    keys = []
    for _ in range(levels):
        k = rng.integers(0, values, size=n_events).astype(np.uint32)
        k[rng.random(n_events) < p_absent] = ABSENT
        keys.append(k)
    letters = rng.integers(0, 1 << atoms, size=n_events).astype(np.uint8)
    return keys, letters


def c5_trace(seed: int = 0, n: int = 2_000_000, hosts: int = 256, users: int = 100_000,
             mean_len: float = 10.0, span_events: int = 2_000_000,
             p=(0.01, 0.3, 0.3, 0.01, 0.05)) -> Trace:
    """C5: three-level keys (host, user, session); sessions are unique with ~mean_len
    events spread over ~span_events positions (about two 1M-event batches).
    Letter bits follow the atom union of C5_FORMULAS: authfail, request, response,
    admin, external."""
    rng = np.random.default_rng(SEED_BASE + 5 + seed)
    S = max(1, int(n / mean_len))
    lens = 1 + rng.poisson(mean_len - 1, size=S)
    starts = rng.random(S) * n
    ev_sess = np.repeat(np.arange(S), lens)
    gaps = rng.exponential(span_events / mean_len, size=ev_sess.shape[0])
    first = np.r_[0, np.cumsum(lens)[:-1]]
    cs = np.cumsum(gaps)
    t = starts[ev_sess] + cs - np.repeat(cs[first], lens)
    order = np.argsort(t, kind="stable")[:n]
    ev_sess = ev_sess[order]
    user_of = rng.integers(0, users, size=S)
    home = rng.integers(0, hosts, size=users)
    roam = rng.random(S) < 0.1
    host_of = np.where(roam, rng.integers(0, hosts, size=S), home[user_of])
    hid, uid, sid = _ids(rng, hosts), _ids(rng, users), _ids(rng, S)
    letters = np.zeros(ev_sess.shape[0], dtype=np.uint8)
    for j, pj in enumerate(p):
        letters |= (rng.random(ev_sess.shape[0]) < pj).astype(np.uint8) << j
    keys = [hid[host_of[ev_sess]], uid[user_of[ev_sess]], sid[ev_sess]]
    return Trace("\n".join(C5_FORMULAS), keys, letters, {"config": "C5", "seed": seed})


def to_jsonl(tr: Trace, key_names, atom_preds, atom_args, seed: int = 0, style: str = "mixed") -> str:
    """Write a trace as JSON-lines key -> value records (the paper's key-value events,
    P:922-925): guard key i -> the event's value (absent keys omitted), 0-ary atom ->
    `true` when it holds, parametric atom q(x_i) -> the event's own value of x_i (or
    `true`).  No method arithmetic: values are formatted, never interpreted.

    style "mixed" writes each value in one of several spellings that denote the same
    value (integer, string, decimal with trailing zeros, exponent) plus noise keys, so
    readers must canonicalise; "plain" writes integers only."""
    import json as _json
    rng = np.random.default_rng(SEED_BASE + 900 + seed)
    n = tr.n
    pick = rng.integers(0, 4, size=(len(key_names), n)) if style == "mixed" else np.zeros((len(key_names), n), int)
    atom_true = rng.random(n) < 0.5
    noise = rng.random(n) < 0.1
    lines = []

    def spell(v: int, how: int):
        if how == 0:
            return str(v)
        if how == 1:
            return _json.dumps(str(v))
        if how == 2:
            return f"{v}.000"
        return f"{v / 10:.1f}e1" if v % 10 == 0 and v else str(v) if v < 10 else f"{v // 10}.{v % 10}e1"

    for j in range(n):
        parts = []
        vals = []
        for i, k in enumerate(key_names):
            v = int(tr.keys[i][j])
            vals.append(None if v == 0xFFFFFFFF else v)
            if v != 0xFFFFFFFF:
                parts.append(f'{_json.dumps(k)}: {spell(v, int(pick[i, j]))}')
        a = int(tr.letters[j])
        for b, (q, args) in enumerate(zip(atom_preds, atom_args)):
            if not (a >> b) & 1:
                continue
            if not args or atom_true[j] or any(vals[x] is None for x in args):
                if args and any(vals[x] is None for x in args):
                    continue  # the atom cannot hold without its argument's value (A12)
                parts.append(f'{_json.dumps(q)}: true')
            elif len(args) == 1:
                parts.append(f'{_json.dumps(q)}: {vals[args[0]]}')
            else:
                parts.append(f'{_json.dumps(q)}: [{", ".join(str(vals[x]) for x in args)}]')
        if noise[j]:
            parts.append('"note": {"level": "info", "tags": ["a", 1, null]}')
        lines.append("{" + ", ".join(parts) + "}")
    return "\n".join(lines) + "\n"
