"""Data-parallel plumbing for the packed hot path ("8-GPU data parallel").

Packed rows are independent units (no sequence spans rows; the reset
cuts every carry), so G GPUs take contiguous blocks of rows and run all four
kernels locally.  The only exchange is one all-reduce (sum) of the flattened
parameter gradients [dA | dD | ddt_bias | dw | dbias] of this path
(SURVEY §8(e)).  dB, dC, du, ddt, dx are per-token and stay local.

torch.distributed is used as plumbing only (NCCL over NVLink on the GPU box,
gloo in the CPU tests).
"""
from __future__ import annotations


def shard_rows(total_rows: int, rank: int, world: int) -> range:
    """Contiguous block of global row ids owned by ``rank``."""
    if total_rows % world:
        raise ValueError(f"{total_rows} rows do not split over {world} ranks")
    per = total_rows // world
    return range(rank * per, (rank + 1) * per)


class ParamGrads:
    """One flat fp32 buffer holding every parameter gradient of the path, so
    the kernels write straight into it and a single all-reduce syncs it."""

    def __init__(self, torch, Dn: int, N: int, K: int, device):
        self.sizes = dict(dA=Dn * N, dD=Dn, ddt_bias=Dn, dw=Dn * K, db=Dn)
        self.shapes = dict(dA=(Dn, N), dD=(Dn,), ddt_bias=(Dn,), dw=(Dn, K), db=(Dn,))
        self.flat = torch.zeros(sum(self.sizes.values()), dtype=torch.float32, device=device)
        self.views = {}
        off = 0
        for k, n in self.sizes.items():
            self.views[k] = self.flat[off:off + n].view(self.shapes[k])
            off += n

    def __getitem__(self, k):
        return self.views[k]

    @property
    def nbytes(self) -> int:
        return self.flat.numel() * 4

    def allreduce(self, dist, group=None) -> None:
        dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=group)
