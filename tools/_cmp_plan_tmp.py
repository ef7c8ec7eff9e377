import sys, os, ctypes, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2502_20766_b200 as fp
import torch
from synth import configs, gen
w = configs.get("C2-llama8b-32k")
qb_, kb_, vb_ = gen.make_layer_bits(w)
q, k, v = (torch.from_numpy(x).view(torch.bfloat16).cuda() for x in (qb_, kb_, vb_))
K = gen.bits_to_f64(kb_)
ref = K.reshape(w.kv_heads, -1, 128, 128).mean(axis=2)
fp.load_library()
for name in sys.argv[1:]:
    L = ctypes.CDLL(os.path.abspath(name), mode=os.RTLD_LOCAL)
    P, I, Z, F = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t, ctypes.c_float
    L.fp_plan.argtypes = [P, P, I, I, I, I, I, F, P, Z, P, P, P]
    f = fp.FlexPrefill(w.heads, w.kv_heads, w.seq_len)
    st = torch.cuda.current_stream().cuda_stream
    f.ws.zero_()
    r = L.fp_plan(q.data_ptr(), k.data_ptr(), w.heads, w.kv_heads, w.seq_len, 128, 128, w.tau,
                  f.ws.data_ptr(), f.ws_bytes, f.pattern.data_ptr(), f.jsd.data_ptr(), st)
    torch.cuda.synchronize()
    kbar = f.debug()["k_bar"].numpy()
    d = np.abs(kbar - ref)
    bad = np.argwhere(d > 1e-3)
    print(name, "k_bar maxdiff", d.max(), "nbad", len(bad), bad[:3].tolist())
