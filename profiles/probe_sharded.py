"""Phase timing of the sharded step (GpuShard + TorchComm/NCCL) at world size 1."""
import os, sys, time, socket
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist
from paper_1411_1702_b200 import problems
from paper_1411_1702_b200.sharded import GpuShard, ShardedFilter, TorchComm, BUF_PRED, BUF_PRED_ALL, BUF_SUM, BUF_SUM_ALL, BUF_HDR, BUF_WIN, BUF_MOM, BUF_MOM_ALL, BUF_CNT, BUF_CNT_ALL, STEP_FLAGS
sk = socket.socket(); sk.bind(("127.0.0.1", 0)); port = sk.getsockname()[1]; sk.close()
torch.cuda.set_device(0)
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1, device_id=torch.device("cuda:0"))
n = 1 << 20
prob = problems.lotka_volterra(particles=n, T=40, seed=1)
s = GpuShard("lv", prob.cfg, prob.obs, 0, 1)
f = ShardedFilter([s], TorchComm())
f.initialize_uniform(**prob.prior)
comm, sh = f.comm, f.shards
tp = 0.0
acc = {}
def T(name, fn):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = fn(); torch.cuda.synchronize()
    acc[name] = acc.get(name, 0.0) + time.perf_counter() - t0
    return r
for j in range(1, 21):
    y, t1 = prob.ys[j - 1], prob.times[j - 1]
    T("predict", lambda: s.predict(y, j, tp, t1, 0.1))
    T("A", lambda: comm.allgather(sh, BUF_PRED, BUF_PRED_ALL))
    T("finish_lse", lambda: s.finish_lse())
    T("B", lambda: comm.allgather(sh, BUF_SUM, BUF_SUM_ALL))
    T("scan_records", lambda: s.scan_records())
    T("C", lambda: (comm.allgather_slices(sh, BUF_HDR), comm.allgather_slices(sh, BUF_WIN)))
    T("resolve", lambda: s.resolve())
    served = T("serve", lambda: {s.rank: s.serve()})
    mat = T("counts", lambda: s.count_matrix())
    counts = {0: mat[0]}
    T("exchange", lambda: comm.exchange(sh, counts, 8 * s.payload_doubles()))
    T("update", lambda: s.update(int(counts[0][0])))
    T("E", lambda: comm.allgather(sh, BUF_MOM, BUF_MOM_ALL))
    T("finish_moments", lambda: s.finish_moments(STEP_FLAGS))
    tp = t1
for k, v in acc.items():
    print(f"{k:15s} {1e3 * v / 20:8.3f} ms")
print("total", 1e3 * sum(acc.values()) / 20)
dist.destroy_process_group()
