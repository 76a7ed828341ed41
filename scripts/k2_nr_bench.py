"""K2 (apply_quant) cost versus rank count on one GPU (development tool): the same
ResNet-50 layout with nranks = 1, 2, 4, 8 gathered code windows, CUDA-event timed."""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2106_10796_b200 import _lib  # noqa: E402
from paper_2106_10796_b200.layout import by_name  # noqa: E402


def timeit(fn, reps=20, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def codes(nw, nr):
    f = torch.randint(0, 3, (nr * nw, 16), device="cuda", dtype=torch.int64)
    sh = 2 * torch.arange(16, device="cuda", dtype=torch.int64)
    return (f << sh).sum(1).to(torch.uint32).view(torch.int32)


def main():
    lay = by_name(sys.argv[1] if len(sys.argv) > 1 else "resnet50")
    n, nw = lay.total, lay.n_words
    lib = _lib.load()
    h = lay.handle().ptr
    st = torch.cuda.current_stream().cuda_stream
    W = torch.randn(n, device="cuda")
    g = torch.randn(n, device="cuda")
    loc = torch.empty(n, device="cuda")
    gn = torch.zeros(1, dtype=torch.float64, device="cuda")
    out = {}
    for nr in (1, 2, 4, 8):
        cw = codes(nw, nr)
        for tag, gp in (("loc", True), ("noloc", False)):
            fn = lambda: lib.cdsgd_apply_quant(h, W.data_ptr(), 0, cw.data_ptr(), nr, nw, 0.5, 0.1,
                                               g.data_ptr() if gp else None, loc.data_ptr() if gp else None, 0.4,
                                               None, 0, gn.data_ptr(), st)
            out[f"nr{nr}_{tag}"] = round(timeit(fn), 1)
    # the same with W and the code windows inside a symmetric-memory allocation (p2p mode)
    if os.environ.get("SYMM") == "1":
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29561")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        nb = 4 * n + 4 * 4 * nw + 4096
        buf = symm_mem.empty(nb, dtype=torch.uint8, device="cuda")
        symm_mem.rendezvous(buf, dist.group.WORLD)
        Ws = buf[: 4 * n].view(torch.float32)
        Ws.copy_(W)
        cs = buf[4 * n: 4 * n + 16 * nw].view(torch.int32)
        cs.copy_(codes(nw, 4))
        for tag, Wp, cp in (("symmW_symmC", Ws, cs), ("symmW_regC", Ws, codes(nw, 4)), ("regW_symmC", W, cs)):
            fn = lambda: lib.cdsgd_apply_quant(h, Wp.data_ptr(), 0, cp.data_ptr(), 4, nw, 0.5, 0.1, g.data_ptr(),
                                               loc.data_ptr(), 0.4, None, 0, gn.data_ptr(), st)
            out[f"nr4_loc_{tag}"] = round(timeit(fn), 1)
        dist.destroy_process_group()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
