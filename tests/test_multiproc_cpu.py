"""World-size-2 gloo tests of the N>1 host path (CPU only, torch.distributed on 127.0.0.1).

* every rank's control plane reaches the identical mode timeline from all-gathered batch sizes,
  equal bit-for-bit to the oracle's policy (oracle/policy.py is separate code);
* every rank's library-built plan/stagger (sidp_init, host only) agrees with the oracle and the
  union over ranks has the single-reader property at every tick.
"""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_28095_b200 import orchestrator as O
        import paper_2605_28095_b200 as P
        from sidp_inputs import MODELS
        # ---- mode control plane: each rank only knows its own batch trace
        traces = {0: [100] * 150 + [3] * 200 + [40] * 150,
                  1: [120] * 150 + [0] * 200 + [10] * 150}
        ctl = O.ModeController(O.ModePolicy(b_threshold=16, window=50, hysteresis=1.5,
                                            min_dwell=100), world)
        modes = [ctl.mode]
        for t in range(len(traces[0])):
            b = O.gather_batches(traces[rank][t], dist)
            modes.append(ctl.observe(b))
        # ---- library schedule per rank (host only, no GPU)
        m = MODELS["tiny"].with_layers(8 * world)
        ctx = P.Context(m, rank=rank, world=world, slots=2, alloc=False)
        info = {"plan": ctx.plan(), "stagger": ctx.stagger_ticks(),
                "owners": [ctx.owner_of(l) for l in range(m.num_layers)]}
        ctx.destroy()
        gathered = [None] * world
        dist.all_gather_object(gathered, {"modes": modes[:-1], "info": info})
        q.put((rank, gathered))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_group_control_plane_gloo(world):
    from paper_2605_28095_b200 import build as B
    B.build()
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle import policy as OP
    from oracle import schedule as OS
    g = res[0]
    assert g == res[1]                                   # identical view on every rank
    modes = [x["modes"] for x in g]
    assert modes[0] == modes[1]                          # globally consistent
    traces = [[100] * 150 + [3] * 200 + [40] * 150, [120] * 150 + [0] * 200 + [10] * 150]
    per_step = [[traces[0][t], traces[1][t]] for t in range(500)]
    ref = OP.mode_timeline(OP.ModePolicy(16, 50, 1.5, 100), per_step)
    assert modes[0] == ref
    assert OP.CAS in ref and ref[-1] == OP.WAS           # tail -> CaS, burst above 24 -> WaS
    # schedule: plans and stagger equal the oracle; single reader at every tick
    L = 8 * world
    own = OS.owner_map(L, world)
    plans = [x["info"]["plan"] for x in g]
    offs = [x["info"]["stagger"] for x in g]
    for r in range(world):
        assert plans[r] == OS.plan_exec(own, r)
        assert offs[r] == OS.stagger_ticks(world, r)
        assert g[r]["info"]["owners"] == own
    assert OS.single_reader_violations(own, world, 4 * len(plans[0]), plans, offs) == 0
