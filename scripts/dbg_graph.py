import sys
sys.path.insert(0, '.')
import torch
from paper_1706_06664_b200 import _native as N, ace, workloads as W
w = W.CONFIGS[5]
for n in (65536*2, 65536*4+1000):
    x = torch.empty((n, w.dim), dtype=torch.float32, device="cuda")
    W.device_rows(5, 0, n, x.data_ptr())
    fam = ace.SrpFamily(ace.SrpConfig(dim=w.dim, k_bits=w.k_bits, num_tables=w.num_tables, seed=w.w_seed))
    for use_torch_stream in (False, True):
        sk = ace.AceSketch(fam, ace.CounterWidth.k32)
        if use_torch_stream:
            sk.set_stream(torch.cuda.current_stream().cuda_stream)
            print("torch stream handle", torch.cuda.current_stream().cuda_stream)
        flags = torch.empty((n + 31) // 32, dtype=torch.int32, device="cuda")
        for i in range(3):
            sk.reset()
            try:
                _, lat, rep = sk.stream_run(x, w.batch, w.alpha, flags_out=flags)
                print(n, use_torch_stream, i, "ok", rep.reported, lat[:3])
            except Exception as e:
                print(n, use_torch_stream, i, "ERR", e)
