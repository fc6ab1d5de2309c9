"""WaS <-> CaS mode switching on virtual ranks: the directive is issued with
identical arguments on every rank, takes effect at a step boundary, drains and resets the WaS
ring, and the decoded sequence equals a replicated run throughout (WaS steps bitwise, CaS steps
within tolerance) and the fp64 oracle's decode of the same tokens (north_star tolerance).  Also
the controller-driven switch: per-step batches gathered on the host feed the orchestrator
policy, whose directive every rank applies."""
import numpy as np
import pytest
import torch

from oracle import model as OM
from oracle import schedule as OS
from sidp_inputs import MODELS

from .test_gpu_parity import SEED, TOL, Rank, _budget, _gpu_caches, _group, _replicated, P  # noqa: F401  (fixture)
from .helpers import OracleModel, oracle_layer, rank_inputs, rel_err

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("pool", ["layer", "ffn"])
def test_was_cas_was_switch(P, pool):
    m = MODELS["tiny"].with_layers(8)
    B = [3, 5]
    ranks = _group(P, m, 2, B, pool=pool)
    for R in ranks:
        R.ctx.set_batches(B)
    schedule = {2: 1, 4: 0}          # step -> mode (1 = CaS, 0 = WaS)
    for s in range(6):
        if s in schedule:
            for R in ranks:
                R.ctx.set_mode(schedule[s], s)
        for R in ranks:
            R.step()
        for R in ranks:
            R.finish_step()
        for R in ranks:
            assert R.ctx.stats()["mode"] == (1 if 2 <= s < 4 else 0)
    for r, R in enumerate(ranks):
        assert R.ctx.stats()["timeouts"] == 0
        rep = _replicated(P, m, B[r], sum(B[:r]), pool=pool, compute_sms=_budget(R))
        for s in range(6):
            rep.toks = R.history[s - 1][0].cuda() if s else rep.toks   # follow the same tokens
            rep.step(); rep.finish_step()
            got, exp = R.history[s][1], rep.history[s][1]
            if s < 2:
                assert torch.equal(got, exp), (r, s)
            else:
                assert rel_err(got.double().numpy(), exp.double().numpy()) <= TOL, (r, s)
        rep.ctx.destroy()
        # and against the fp64 ORACLE through the whole WaS -> CaS -> WaS run (not only against
        # another GPU run), per layer as the north_star states its tolerance: every step's every
        # layer recomputed by the oracle from the GPU's bf16 layer input and KV state (teacher
        # forcing; the oracle's CaS layer equals its replicated layer to 1e-12,
        # tests/test_oracle_model.py), against the next layer's input, the new k/v entries at
        # pos + s and the logits
        om = OracleModel(m, SEED)
        _, _, pos, _ = rank_inputs(m, SEED, sum(B[:r]), B[r], 0, 63, 80)
        Kg, Vg = _gpu_caches(R, B[r])
        b = np.arange(B[r])
        for s in range(6):
            _, logits, dump = R.history[s]
            xs = dump.double().numpy()
            for l in range(m.num_layers):
                out, kn, vn = oracle_layer(om, l, xs[l], pos + s, Kg[l], Vg[l])
                errs = [rel_err(Kg[l][b, pos + s], kn), rel_err(Vg[l][b, pos + s], vn)]
                if l + 1 < m.num_layers:
                    errs.append(rel_err(xs[l + 1], out))
                else:
                    errs.append(rel_err(logits.double().numpy(), OM.lm_head(m, om.head, out)))
                assert max(errs) <= TOL, (r, s, l, errs)
        # after the switch back the ring restarted: the log tail is a fresh FIFO schedule
        own = OS.owner_map(8, 2)
        log = R.ctx.fetch_log()
        ref = OS.slot_schedule(OS.plan_exec(own, r), 2, 3)
        assert log == ref[:len(log)]
    for R in ranks:
        R.ctx.destroy()


def test_controller_driven_switch(P):
    """The orchestrator decides from gathered batch sizes; every rank gets the same directive."""
    from paper_2605_28095_b200.orchestrator import ModeController, ModePolicy
    m = MODELS["tiny"].with_layers(4)
    B = [4, 2]
    ranks = _group(P, m, 2, B)
    ctl = ModeController(ModePolicy(b_threshold=8, window=2, hysteresis=1.5, min_dwell=2), world=2)
    modes = []
    for s in range(6):
        for R in ranks:
            R.ctx.set_batches(B)
        for R in ranks:
            R.step()
        for R in ranks:
            R.finish_step()
        nxt = ctl.observe(B)                        # both ranks see the same gathered batches
        for R in ranks:
            R.ctx.set_mode(nxt, s + 1)
        modes.append([R.ctx.stats()["mode"] for R in ranks])
    assert all(a == b for a, b in modes)            # globally consistent
    assert modes[0] == [0, 0] and modes[-1] == [1, 1]
    for R in ranks:
        assert R.ctx.stats()["timeouts"] == 0
        R.ctx.destroy()


def test_cas_peer_timeout_surfaces_etimeout(P, monkeypatch):
    """A CaS peer that never arrives: the owner's device-side flag wait gives up after
    SIDP_CAS_TIMEOUT_MS, writes the mapped host error word, and every later call on that
    context returns SIDP_ETIMEOUT (sidp.h); sidp_stats counts it."""
    monkeypatch.setenv("SIDP_CAS_TIMEOUT_MS", "200")
    m = MODELS["tiny"].with_layers(2)
    ranks = _group(P, m, 2, [2, 2])
    for R in ranks:
        R.ctx.set_batches([2, 2])
        R.ctx.set_mode(1, 0)
    R = ranks[0]
    x = torch.zeros(2, m.hidden, dtype=torch.bfloat16, device="cuda")
    R.ctx.decode_layer(x, 0, 1, R.kv, batch=2, stream=R.stream)   # rank 1 never calls
    R.stream.synchronize()
    with pytest.raises(P.SidpError) as e:
        R.ctx.decode_layer(x, 1, 1, R.kv, batch=2, stream=R.stream)
    assert e.value.status == -6
    assert R.ctx.stats()["timeouts"] >= 1
    for Q in ranks:
        Q.ctx.destroy()
