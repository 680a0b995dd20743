"""sharded_batch_counts under torch.distributed (2 ranks on one GPU, gloo
backend: the NCCL path needs one GPU per rank) against batch_counts:
   torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/sharded_check.py"""
import os, sys
import numpy as np
import torch
import torch.distributed as dist
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1711_03637_b200 as sd  # noqa: E402
from paper_1711_03637_b200 import distributed as sdist  # noqa: E402
dist.init_process_group("gloo")
torch.cuda.set_device(0)
d = np.load(os.path.join(ROOT, "data", "workloads.npz"))
w = np.load(os.path.join(ROOT, "data", "w_fix.npz"))["w_fix"]
imgs = d["c3_images"][:2000]
cfg, bank = sd.NetworkConfig(), sd.default_filter_bank()
got = sdist.sharded_batch_counts(imgs, w, bank, cfg)
want = sd.batch_counts(imgs, w, bank, cfg)
ok = got.dtype == np.int64 and np.array_equal(got, want)
print(f"rank {dist.get_rank()}: sharded == batch_counts: {ok}", flush=True)
dist.destroy_process_group()
sys.exit(0 if ok else 1)
