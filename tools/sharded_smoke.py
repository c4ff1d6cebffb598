"""Sharded (NCCL) device path at world size 1 under torchrun (GPU box):
    python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
        --master-port 29511 tools/sharded_smoke.py
LINKCERT_FORCE_SHARDED=1 routes certificates through the library's own NCCL
communicator (lc_comm_init + lc_run_pipeline_sharded: cost-balanced item range,
in-place MAX all-reduce, fixed-order reduce); results must equal the unsharded
path bitwise."""
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
from paper_2106_12655_b200.certify import run_device_pipeline
print("nccl version (library-loaded):", _native.nccl_version(), flush=True)
cases = {"kusari_small": (gen.kusari_tube(n_around=12, rows=4, partial=5),
                          gen.kusari_tube(n_around=12, rows=4, partial=5), lc.KernelChoice()),
         # long loops: the staged sharded path (cost-balanced gauss_run range + all-reduce)
         "knit_4x2000": (gen.knit_tube(courses=4, n=2000, W=10), gen.knit_tube(courses=4, n=2000, W=10),
                         lc.KernelChoice()),
         "kusari_small_anglesum": (gen.kusari_tube(n_around=12, rows=4, partial=5),
                                   gen.kusari_tube(n_around=12, rows=4, partial=5),
                                   lc.KernelChoice(ds_variant="anglesum"))}
for name, (before, after, choice) in cases.items():
    cert = lc.compute_linking_matrix(before, choice=choice)
    path = _native.context().last_run_fused()
    sharded = [np.array(a).copy() for a in run_device_pipeline(before, mode=lc.direct.ds_mode(choice.ds_variant))[:4]]
    os.environ["LINKCERT_FORCE_SHARDED"] = "0"
    want = lc.compute_linking_matrix(before, choice=choice)
    plain = [np.array(a).copy() for a in run_device_pipeline(before, mode=lc.direct.ds_mode(choice.ds_variant))[:4]]
    os.environ["LINKCERT_FORCE_SHARDED"] = "1"
    assert cert.entries == want.entries and cert.model_digest == want.model_digest, name
    for a, b in zip(sharded, plain):
        assert np.array_equal(a, b), name          # bitwise, raw sums included
    for _ in range(3):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            rep = lc.verify(after, cert, choice=choice)
    print(name, "sharded path", path, "->", _native.context().last_run_fused(), rep.status, len(cert.entries), flush=True)
dist.destroy_process_group()
print("sharded smoke ok")
