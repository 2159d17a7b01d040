import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import oracle, tracegen, paper_1411_2239_b200 as ltl4c
dev = torch.device('cuda:0')
for n, videos in [(20_000, 500), (100_000, 2000), (300_000, 5000), (1_000_000, 20_000)]:
    tr = tracegen.proxy_trace(seed=3, n=n, videos=videos, p_ext_cached=0.002)
    st = ltl4c.compile(tr.formula).state(0)
    st.profile(True)
    k = [torch.from_numpy(x.view(np.int32)).to(dev) for x in tr.keys]
    l = torch.from_numpy(tr.letters).to(dev)
    t = time.time()
    r = st.verify(k, l)[0]
    el = time.time() - t
    w = oracle.run_offline(tr.formula, tr.keys, tr.letters)
    print(n, videos, f"{el:.3f}s", r.verdict, w['verdict'], np.array_equal(r.hist, w['hist']), st.stats()['kernels']['bucket_global'], flush=True)
