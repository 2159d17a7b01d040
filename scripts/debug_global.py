import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import oracle, tracegen, paper_1411_2239_b200 as ltl4c
dev = torch.device('cuda:0')
case = sys.argv[1]
def run(text, keys, letters, online):
    st = ltl4c.compile(text).state(0, online=online)
    k = [torch.from_numpy(np.ascontiguousarray(x).view(np.int32)).to(dev) for x in keys]
    t = time.time()
    r = st.verify(k, torch.from_numpy(letters).to(dev))[0]
    w = oracle.run_offline(text, keys, letters)
    print(case, f"{time.time()-t:.3f}s", r.verdict, w['verdict'], np.array_equal(r.hist, w['hist']), flush=True)
if case == 'c4_online':
    tr = tracegen.proxy_trace(seed=3, n=20_000, videos=500); run(tr.formula, tr.keys, tr.letters, True)
if case == 'c4_offline':
    tr = tracegen.proxy_trace(seed=3, n=20_000, videos=500); run(tr.formula, tr.keys, tr.letters, False)
if case == 'c2_online':
    tr = tracegen.login_trace(seed=3, n=20_000, users=50, rid_events=2); run(tr.formula, tr.keys, tr.letters, True)
if case == 'sock_offline_big':
    tr = tracegen.socket_trace(seed=0, n=10_000, sockets=3); run(tr.formula, tr.keys, tr.letters, False)
if case == 'login_2users':
    tr = tracegen.login_trace(seed=3, n=5000, users=2); run(tr.formula, tr.keys, tr.letters, False)
