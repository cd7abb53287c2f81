"""Can torch capture an NCCL all_to_all_single inside a CUDA graph on this image?
(single-rank NCCL group; the prerequisite for graph replay of the sequence-parallel loop)"""
import os

import torch
import torch.distributed as dist

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29555")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
send = torch.randn(4, 1024, device="cuda", dtype=torch.bfloat16)
recv = torch.empty_like(send)
dist.all_to_all_single(recv, send)  # eager warm-up (communicator init)
torch.cuda.synchronize()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(2):
        dist.all_to_all_single(recv, send * 2)
torch.cuda.current_stream().wait_stream(s)
g = torch.cuda.CUDAGraph()
try:
    with torch.cuda.graph(g):
        tmp = send * 3
        dist.all_to_all_single(recv, tmp)
    send.copy_(torch.randn_like(send))
    g.replay()
    torch.cuda.synchronize()
    ok = torch.equal(recv, send * 3)
    print("captured all_to_all_single in a CUDA graph; replay correct:", ok)
except Exception as e:  # report, do not crash
    print("capture failed:", repr(e)[:300])
dist.destroy_process_group()
