"""Host-side multi-rank logic on CPU (no GPU):

* PP send/recv pairing (north_star invariant "stage send/recv pairing"): for
  every virtual-stage edge (src vs -> dst vs, forward or backward) the k-th
  PP_SEND on that edge carries the same microbatch as the k-th PP_RECV.  This
  FIFO property is what lets the executor use one unidirectional NCCL
  communicator + stream per edge.  (One channel per device PAIR is not
  enough: ZB and 1F1B-I interleave forward and backward messages on a pair in
  different orders at the two ends — test_device_pair_channel_is_not_fifo.)
* The product's parameter packer (stage.pack_rank_param) vs the oracle's
  independent shard_params for every TP rank.
* A world_size-2 gloo process group: NCCL-id broadcast (the rendezvous the
  stage uses) and rank -> (tp_rank, pp_rank) mapping, exercised with real
  torch.distributed collectives.
"""
import dataclasses
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import stp_inputs as si
from oracle import model as om
from oracle import schedule as sc


def _link_sequences(kind, p, m, lay):
    progs = sc.build_program(kind, p, m)
    V = sc.n_vstages(kind, p)
    sends, recvs = {}, {}
    for d in range(p):
        units = sc.expand_units(kind, p, d, progs[d], lay)
        for u in units:
            ai, stream, op, peer, c, mb, d0, d1 = u
            vs = sc.vstage(kind, p, d, c)
            if op == sc.PP_SEND:
                fwd = units[d0][2] == sc.CF
                dst_vs = vs + 1 if fwd else vs - 1
                sends.setdefault((d, peer), []).append((mb, vs, dst_vs))
            elif op == sc.PP_RECV:
                j = units.index(u)
                fwd = any(v[2] == sc.CF and v[6] == j for v in units)
                src_vs = vs - 1 if fwd else vs + 1
                recvs.setdefault((peer, d), []).append((mb, src_vs, vs))
    return sends, recvs, V


@pytest.mark.parametrize("kind", [sc.STP, sc.STP_NOSEP, sc.ONEF1B_I, sc.ZB, sc.ONEF1B])
@pytest.mark.parametrize("p", [2, 3, 4])
def test_pp_links_are_fifo(kind, p):
    for m in (p, 2 * p, 4 * p):
        if kind == sc.ONEF1B_I and m % p:
            continue
        lay = [1] * sc.n_vstages(kind, p)
        sends, recvs, _ = _link_sequences(kind, p, m, lay)
        assert set(sends) == set(recvs)
        for link in sends:
            edges = {(e[1], e[2]) for e in sends[link]}
            for edge in edges:
                a = [e[0] for e in sends[link] if (e[1], e[2]) == edge]
                b = [e[0] for e in recvs[link] if (e[1], e[2]) == edge]
                assert a == b == list(range(1, m + 1)), (link, edge)
            assert sorted(sends[link]) == sorted(recvs[link])


def test_device_pair_channel_is_not_fifo():
    sends, recvs, _ = _link_sequences(sc.ZB, 2, 4, [1, 1, 1, 1])
    assert any(sends[k] != recvs[k] for k in sends)


@pytest.mark.parametrize("t", [1, 2, 4])
def test_product_packer_matches_oracle_shards(t):
    from paper_2510_27257_b200.stage import pack_rank_param
    cfg = dataclasses.replace(si.TINY, n_kv_heads=4)
    P = si.make_params(cfg, seed=4, parity=True)
    for r in range(t):
        ref = om.shard_params(P, cfg, t, r)
        for name, arr in ref.items():
            assert np.array_equal(pack_rank_param(name, P, cfg, t, r), arr), (t, r, name)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2510_27257_b200.stage import broadcast_nccl_id
    uid = broadcast_nccl_id()
    # grid mapping used by bench.py / the stage: rank = pp_rank * tp + tp_rank
    import bench
    t, p = bench.CONFIGS["cfg2"][3][world]
    got = [None] * world
    dist.all_gather_object(got, (rank % t, rank // t, uid))
    q.put((rank, got))
    dist.destroy_process_group()


def test_gloo_world2_rendezvous():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, got in res:
        assert [g[:2] for g in got] == [(0, 0), (1, 0)]      # tp=2, pp=1 at world 2
        ids = {g[2] for g in got}
        assert len(ids) == 1 and len(next(iter(ids))) == 128  # one ncclUniqueId, 128 bytes
