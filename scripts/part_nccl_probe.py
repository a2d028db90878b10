import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.getcwd())
import paper_1908_00210_b200 as pi
from paper_1908_00210_b200 import sharding as sh
def tparams(s):
    p = pi.AnnealParams(); p.sweeps, p.workers = s, 8; return p
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
pi.set_device(0)
g = pi.random_graph(100000, 400000, 77)
prob = pi.MinCutProblem.with_default_coefficients(g)
for seed in (5, 6, 7):
    pa = sh.PartitionedAnneal(prob, tparams(30), seed, dist, 0)
    for k in range(2):
        r = pa.run()
        print(os.environ.get("GDI_K4_FRAC"), seed, k, r["cut"], r["imbalance"], r["balance_counter"], int(r["spins"].astype(np.int64).sum()), flush=True)
    pa.close()
dist.destroy_process_group()
