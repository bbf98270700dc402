"""Cross-process exchange of the per-round bound (multi-GPU).

One process per GPU.  Each rank enumerates its shard of every round
(``bz_round(..., shard=rank, nshards=world)``: chunk c of the round's work
plan belongs to rank c % world) and the ranks then combine one vector of m
per-Gamma minima by MIN and m combination counters by SUM -- one
collective per round over NCCL/NVLink (an all-gather of 2m int64, reduced
locally; gloo on CPU for the tests).  This is
the only exchange the path has; the reference itself is
single-process (enumeration.py:385-444 uses threads).
"""

from __future__ import annotations


class LocalComm:
    """Single process: nothing to exchange."""

    rank = 0
    world = 1

    def combine(self, mins: list[int], combos: list[int]):
        return list(mins), list(combos)

    def barrier(self) -> None:
        pass

    def broadcast_bytes(self, data: bytes | None, src: int = 0) -> bytes | None:
        return data


class TorchComm:
    """torch.distributed default group (nccl on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist

        if not dist.is_initialized():
            raise RuntimeError("torch.distributed is not initialised")
        self._torch = torch
        self._dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        backend = dist.get_backend(group)
        if backend == "nccl":
            self.device = torch.device("cuda", torch.cuda.current_device())
        else:
            self.device = torch.device("cpu")

    def combine(self, mins: list[int], combos: list[int]):
        torch, dist = self._torch, self._dist
        if self.world == 1:
            return list(mins), list(combos)
        m = len(mins)
        width = m + len(combos)  # minima, then the summed counts
        mine = torch.tensor(list(mins) + list(combos), dtype=torch.int64,
                            device=self.device)
        if self.device.type == "cuda":
            allv = torch.empty(self.world * width, dtype=torch.int64, device=self.device)
            dist.all_gather_into_tensor(allv, mine, group=self.group)
            allv = allv.view(self.world, width)
        else:
            parts = [torch.empty_like(mine) for _ in range(self.world)]
            dist.all_gather(parts, mine, group=self.group)
            allv = torch.stack(parts)
        out_min = allv[:, :m].min(dim=0).values.tolist()
        out_sum = allv[:, m:].sum(dim=0).tolist()
        return [int(v) for v in out_min], [int(v) for v in out_sum]

    def barrier(self) -> None:
        self._dist.barrier(group=self.group)

    def broadcast_bytes(self, data: bytes | None, src: int = 0) -> bytes:
        """Rank src's bytes on every rank."""
        obj = [data if self.rank == src else None]
        self._dist.broadcast_object_list(obj, src=src, group=self.group)
        return obj[0]


def combine_rounds(comm, res):
    """Combine several rounds' per-rank (mins, combos) with ONE exchange:
    the vectors are concatenated, reduced (min / sum) and split again."""
    if comm.world == 1 or not res:
        return [(list(mn), list(cb)) for mn, cb in res]
    m = len(res[0][0])
    c = len(res[0][1])  # counts per round (m combinations, or more counters)
    mins, combos = comm.combine([v for mn, _ in res for v in mn],
                                [v for _, cb in res for v in cb])
    return [(mins[i * m:(i + 1) * m], combos[i * c:(i + 1) * c]) for i in range(len(res))]

