import sys, numpy as np, torch
sys.path.insert(0, '.')
import tracegen, paper_1411_2239_b200 as ltl4c
cfg = sys.argv[1]
tr = {"C3": lambda: tracegen.zipf_socket_trace(seed=0),
      "C4": lambda: tracegen.proxy_trace(seed=0, n=125_000_000),
      "C2": lambda: tracegen.login_trace(seed=0)}[cfg]()
dev = torch.device('cuda:0')
k = [torch.from_numpy(x.view(np.int32)).to(dev) for x in tr.keys]
l = torch.from_numpy(tr.letters).to(dev)
st = ltl4c.compile(tr.formula).state(0)
for i in range(2):
    r = st.verify(k, l)[0]
torch.cuda.synchronize()
print("done", r.verdict)
