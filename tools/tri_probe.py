import time, ctypes as C, numpy as np, torch, os, sys
sys.path.insert(0, '/root/repo')
from paper_2602_20826_b200 import _lib, _abi
b = _lib.Corpus(1000000, pinned=True, seed=1).batch()
pin = lambda n, dt: torch.empty(n, dtype=dt, pin_memory=True).numpy()
L = _lib.lib(); pl = _lib.platform(148)
st = pin(b.n_dags, torch.int32); bo = pin(b.n_dags * 10, torch.int64); ng = pin(b.n_dags, torch.int16)
r = _abi.ds_results(st.ctypes.data, bo.ctypes.data, ng.ctypes.data)
ao = b.tri_words(); l16 = pin(b.load_num.shape[0], torch.int16).view(np.uint16); adj = pin(int(ao[-1]), torch.int32).view(np.uint32)
l16, ao_np, adj = b.tri(out=(l16, adj)); ao = pin(ao_np.shape[0], torch.int32).view(np.uint32); ao[:] = ao_np
ct = b.as_ctri(l16, ao, adj)
p16 = (pin(b.load_num.shape[0], torch.int16).view(np.uint16), pin(b.edges.shape[0], torch.int16).view(np.uint16))
a16, e16 = b.compact16(out=p16); c16 = b.as_c16(a16, e16)
def t(f, k=10):
    f(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(k): f()
    return (time.perf_counter() - t0) / k * 1e3
print(os.environ.get('DS_CHUNKS'), os.environ.get('DS_STREAMS'),
      'tri ms', t(lambda: L.ds_analyze_batch_tri(C.byref(ct), C.byref(pl), 0x1F, C.byref(r), 0)),
      '16 ms', t(lambda: L.ds_analyze_batch16(C.byref(c16), C.byref(pl), 0x1F, C.byref(r), 0)))
