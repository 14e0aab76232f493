"""One rank of a multi-GPU solve (launched by tests/test_multigpu.py through
torch.distributed.run): every rank solves the same inputs through
brgpu_create_distributed (NCCL broadcast + all-gathers of the root-range split)
and rank 0 writes the eigenvalues for the single-GPU comparison."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2605_26599_b200 as br  # noqa: E402
from paper_2605_26599_b200 import generators as G  # noqa: E402

out = Path(sys.argv[1])
rank = int(os.environ["RANK"])
dev = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
res = {}
for split in (True, False):
    s = br.distributed_solver(dev, br.BrOptions(root_split=split))
    for fam, n in [("sym-uniform", 1 << 16), ("toeplitz121", 1 << 14), ("wilkinson", 1 << 15), ("sym-uniform", 100001)]:
        d, e = G.generate(fam, n)
        w = s.eigvals(d, e)
        res[f"{fam}_{n}_{int(split)}"] = w
    s.close()
dist.barrier()
if rank == 0:
    np.savez(out, **res)
dist.destroy_process_group()
