"""Multi-process path on CPU: world_size 2 over gloo.  Each rank runs the
real engine loop with EngineConfig(distributed=True) and enumerates only
its shard of every round -- chunks c with c % world == rank of the device
work plan (bz_plan) -- by walking that plan with the oracle; the ranks then
combine through parallel.TorchComm (one all-gather per round).  The result
must equal the reference's trace for the code."""

from __future__ import annotations

import json
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, rows_hex, n, out_path):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                      RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist

    from oracle import oracle
    from paper_1603_06757_b200 import BitMatrix, EngineConfig, _native, engine, minimum_distance

    dist.init_process_group("gloo", rank=rank, world_size=world)

    class ShardRounds:
        def __init__(self, config, comm):
            self.comm = comm

        def load(self, gs, n_):
            self.gammas = [list(gm.rows) for gm in gs.gammas]
            self.k = gs.gammas[0].num_rows

        def run(self, g, lower_prev, upper):
            groups, nchunks = _native.plan(len(self.gammas), self.k, g,
                                           nshards=self.comm.world)
            mins, combos, _ = oracle.enumerate_chunks(self.gammas, self.k, g, groups,
                                                      nchunks, self.comm.rank,
                                                      self.comm.world)
            mins = [upper if v is None else min(v, upper) for v in mins]
            mins, combos = self.comm.combine(mins, combos)
            return mins, combos, 0.0

        def shard(self, g, upper):
            groups, nchunks = _native.plan(len(self.gammas), self.k, g,
                                           nshards=self.comm.world)
            mins, combos, _ = oracle.enumerate_chunks(self.gammas, self.k, g, groups,
                                                      nchunks, self.comm.rank,
                                                      self.comm.world)
            return [upper if v is None else min(v, upper) for v in mins], combos

    class BatchShardRounds(ShardRounds):
        """Adds the batched seam: every round of the batch sharded, one
        exchange for the whole batch (parallel.combine_rounds)."""

        def run_batch(self, g0, lower_prevs, upper):
            from paper_1603_06757_b200.parallel import combine_rounds

            res = [self.shard(g0 + i, upper) for i in range(len(lower_prevs))]
            return combine_rounds(self.comm, res), 0.0

    batched = os.environ.get("BZ_TEST_BATCHED") == "1"
    engine.make_backend = lambda cfg, comm: (BatchShardRounds if batched else ShardRounds)(
        cfg, comm)
    G = BitMatrix([int(r, 16) for r in rows_hex], n)
    cfg = EngineConfig(distributed=True, batch_combinations=10**9 if batched else 0)
    rep = minimum_distance(G, cfg)
    with open(f"{out_path}.{rank}", "w") as fh:
        json.dump(dict(distance=rep.distance, trace=rep.bounds_trace,
                       combos=rep.counters.combinations), fh)
    dist.destroy_process_group()


@pytest.mark.parametrize("batched", [False, True])
@pytest.mark.parametrize("src", ["random_systematic_matrix(9,24,16)",
                                 "random_systematic_matrix(8,26,9)",
                                 "hamming74"])
def test_two_rank_engine(goldens, tmp_path, monkeypatch, src, batched):
    fx = [c for c in goldens["small"]["codes"] if c["src"] == src]
    if not fx:
        fx = [dict(rows=e["rows"], n=e["n"], src=e["src"]) for e in goldens["small"]["enum"]
              if e["src"] == src]
        from oracle import oracle
        rows = [int(r, 16) for r in fx[0]["rows"]]
        ref = oracle.minimum_distance(rows, fx[0]["n"])
        fx[0].update(distance=ref["distance"], bounds_trace=ref["bounds_trace"])
    fx = fx[0]
    out = str(tmp_path / "res")
    monkeypatch.setenv("BZ_TEST_BATCHED", "1" if batched else "0")
    mp.start_processes(_worker, args=(2, _free_port(), fx["rows"], fx["n"], out),
                       nprocs=2, join=True, start_method="spawn")
    res = [json.load(open(f"{out}.{r}")) for r in range(2)]
    for r in res:
        assert r["distance"] == fx["distance"]
        assert [tuple(t) for t in r["trace"]] == [tuple(t) for t in fx["bounds_trace"]]
    assert res[0]["combos"] == res[1]["combos"]
