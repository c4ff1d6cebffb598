"""Sharded (NCCL) device path at world size 1 under torchrun (GPU box):
    python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
        --master-port 29511 tools/sharded_smoke.py
LINKCERT_FORCE_SHARDED=1 routes through the async fused shard run + NCCL MAX all-reduce + reduce."""
import os, sys, warnings
os.environ["LINKCERT_FORCE_SHARDED"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0"))))
import paper_2106_12655_b200 as lc
from paper_2106_12655_b200 import _native, generators as gen
cases = {"kusari_small": (gen.kusari_tube(n_around=12, rows=4, partial=5),
                          gen.kusari_tube(n_around=12, rows=4, partial=5)),
         # long loops: the staged sharded path (gauss_run item ranges + all-gather)
         "knit_4x2000": (gen.knit_tube(courses=4, n=2000, W=10), gen.knit_tube(courses=4, n=2000, W=10))}
for name, (before, after) in cases.items():
    cert = lc.compute_linking_matrix(before)
    path = _native.context().last_run_fused()
    os.environ["LINKCERT_FORCE_SHARDED"] = "0"
    want = lc.compute_linking_matrix(before)
    os.environ["LINKCERT_FORCE_SHARDED"] = "1"
    assert cert.entries == want.entries, name
    for _ in range(3):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            rep = lc.verify(after, cert)
    print(name, "sharded path", path, "->", _native.context().last_run_fused(), rep.status, len(cert.entries), flush=True)
dist.destroy_process_group()
print("sharded smoke ok")
