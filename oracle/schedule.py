"""Integer schedule of SiDP's WaS mode (oracle; test infrastructure only).

Citations are PAPER.md / SPEC.md line numbers plus the section they fall in.
Readings where the paper is silent are SURVEY.md §8(c) C-A* and are listed in
DESIGN.md §3.
"""
from __future__ import annotations

import heapq
import random
from dataclasses import dataclass


# --------------------------------------------------------------------------
# C-S1 owner map — PAPER.md:182 (§4.2 "assign layer (l) to a single owner rank
# r(l)"); rule l mod d from SPEC.md:350-353 (owner_of) — reading C-A1.
# --------------------------------------------------------------------------
def owner_map(num_layers: int, d: int, layer_owner=None) -> list[int]:
    if num_layers < 1 or d < 1:
        raise ValueError("num_layers and d must be >= 1")
    if layer_owner is None:
        return [l % d for l in range(num_layers)]
    owners = list(layer_owner)
    if len(owners) != num_layers:
        raise ValueError("layer_owner must have one entry per layer")
    for o in owners:  # "each layer has exactly one owner"
        if not (0 <= int(o) < d):
            raise ValueError(f"owner {o} not in [0, {d})")
    return [int(o) for o in owners]


# --------------------------------------------------------------------------
# C-S2 plans for one forward pass of rank r.
# --------------------------------------------------------------------------
def plan_exec(owner: list[int], r: int) -> list[int]:
    """Execution order: every non-owned layer, ascending (the north_star's
    "fetch for layer l+1 overlaps layer l"; PAPER.md:188 lookahead of the
    next few layers)."""
    return [l for l, o in enumerate(owner) if o != r]


def peak_shift_order(r: int, c: int, d: int, num_layers: int, owner: list[int]) -> list[int]:
    """One d-layer cycle starting at c: begin at c+r and wrap within the cycle,
    skipping owned layers — PAPER.md:200 (§4.2 Peak shifting).
    A truncated last cycle of width w < d starts at r if r < w else at its
    first layer."""
    w = min(d, num_layers - c)
    start = r if r < w else 0
    seq = [c + ((start + k) % w) for k in range(w)]
    return [l for l in seq if owner[l] != r]


def plan_paper(owner: list[int], d: int, r: int) -> list[int]:
    """Concatenation of peak_shift_order over cycles c = 0, d, 2d, ...
    (SPEC.md:368-376 build_prefetch_plan)."""
    L = len(owner)
    out: list[int] = []
    for c in range(0, L, d):
        out.extend(peak_shift_order(r, c, d, L, owner))
    return out


def plan(owner: list[int], d: int, r: int, order: str) -> list[int]:
    if order == "exec":
        return plan_exec(owner, r)
    if order == "paper":
        return plan_paper(owner, d, r)
    raise ValueError(order)


def fetch_sequence(pl: list[int], steps: int) -> list[tuple[int, int]]:
    """Run-level fetch sequence: the per-pass plan repeated; weights are
    re-fetched every pass (reading C-A7)."""
    return [(t, l) for t in range(steps) for l in pl]


def compute_sequence(pl: list[int], steps: int) -> list[tuple[int, int]]:
    """C-S3: remote (t, l) in the order compute consumes them (ascending l)."""
    remote = sorted(pl)
    return [(t, l) for t in range(steps) for l in remote]


# --------------------------------------------------------------------------
# C-S4 deadlock-freedom (derived).  Fetch j needs the j-th push of the slot
# free-list; S pushes exist initially, then one per completed remote compute.
# --------------------------------------------------------------------------
def lag(pl: list[int]) -> int:
    """max over remote entries of (fetch index p - compute index q) in one pass."""
    q_of = {l: q for q, l in enumerate(sorted(pl))}
    return max((p - q_of[l] for p, l in enumerate(pl)), default=0)


def deadlock_free(pl: list[int], slots: int) -> bool:
    return lag(pl) < slots


# --------------------------------------------------------------------------
# C-S5 slot assignment by FIFO free-list (reading C-A5 of "reserves one slot",
# PAPER.md:193).  Pure recurrence:
#   push[0..S-1] = 0..S-1;  slot(fetch j) = push[j];
#   push[S+k]    = slot of the k-th remote compute entry.
# --------------------------------------------------------------------------
def slot_schedule(pl: list[int], slots: int, steps: int) -> list[tuple[int, int, int]]:
    """Returns [(t, layer, slot)] in fetch order.  Raises if the plan deadlocks."""
    if slots < 1:
        raise ValueError("slots must be >= 1")
    if not deadlock_free(pl, slots):
        raise ValueError("plan deadlocks with this many slots (C-S4)")
    fetches = fetch_sequence(pl, steps)
    computes = compute_sequence(pl, steps)
    p_of = {fk: j for j, fk in enumerate(fetches)}
    push = list(range(slots))
    slot_of_fetch: list[int] = []
    for j in range(len(fetches)):
        while len(push) <= j:
            k = len(push) - slots              # k-th remote compute releases its slot
            push.append(slot_of_fetch[p_of[computes[k]]])
        slot_of_fetch.append(push[j])
    return [(t, l, s) for (t, l), s in zip(fetches, slot_of_fetch)]


# --------------------------------------------------------------------------
# C-S6 explicit event replay of the slot state machine
# Free -> Reserved -> Filling -> Ready -> InUse -> Free.
# Independent of slot_schedule: a discrete-event simulation with real timings.
# --------------------------------------------------------------------------
@dataclass
class ReplayResult:
    completed: bool
    assignments: list           # [(t, layer, slot)] in fetch-issue order
    max_busy: int               # max slots not Free at any instant
    transitions_ok: bool
    consumed_tags_ok: bool


def event_replay(owner: list[int], r: int, pl: list[int], slots: int, steps: int,
                 fetch_time=1.0, compute_time=0.5, jitter=0.0, seed=0,
                 max_events=10**6) -> ReplayResult:
    rng = random.Random(seed)
    fetches = fetch_sequence(pl, steps)
    free = list(range(slots))          # FIFO free-list
    state = ["Free"] * slots
    tag = [None] * slots
    ok_trans = True
    ok_tags = True
    legal = {("Free", "Reserved"), ("Reserved", "Filling"), ("Filling", "Ready"),
             ("Ready", "InUse"), ("InUse", "Free")}

    def move(s, new):
        nonlocal ok_trans
        if (state[s], new) not in legal:
            ok_trans = False
        state[s] = new

    def dur(base):
        return base * (1.0 + jitter * rng.random())

    order = [(t, l) for t in range(steps) for l in range(len(owner))]
    ev = []  # (time, seq, kind, payload)
    seq = 0
    now = 0.0
    nf = 0                  # next fetch index
    fetch_busy = False
    ready_at: dict = {}     # (t,l) -> slot once Ready
    slot_of: dict = {}
    assignments = []
    ci = 0                  # compute cursor into order
    computing = False
    max_busy = 0

    def try_issue_fetch():
        nonlocal nf, fetch_busy, seq
        if fetch_busy or nf >= len(fetches) or not free:
            return
        s = free.pop(0)
        move(s, "Reserved")
        key = fetches[nf]
        tag[s] = key
        slot_of[key] = s
        assignments.append((key[0], key[1], s))
        move(s, "Filling")
        heapq.heappush(ev, (now + dur(fetch_time), seq, "fetched", (key, s)))
        seq += 1
        nf += 1
        fetch_busy = True

    def try_compute():
        nonlocal ci, computing, seq, ok_tags
        while not computing and ci < len(order):
            t, l = order[ci]
            if owner[l] == r:
                ci += 1
                heapq.heappush(ev, (now + dur(compute_time), seq, "owned_done", None))
                seq += 1
                computing = True
                return
            key = (t, l)
            if key not in ready_at:
                return
            s = ready_at.pop(key)
            if tag[s] != key:
                ok_tags = False
            move(s, "InUse")
            ci += 1
            heapq.heappush(ev, (now + dur(compute_time), seq, "remote_done", (key, s)))
            seq += 1
            computing = True
            return

    try_issue_fetch()
    try_compute()
    n_ev = 0
    while ev and n_ev < max_events:
        now, _, kind, payload = heapq.heappop(ev)
        n_ev += 1
        if kind == "fetched":
            key, s = payload
            move(s, "Ready")
            ready_at[key] = s
            fetch_busy = False
        elif kind == "remote_done":
            key, s = payload
            move(s, "Free")       # housekeeper releases after compute completes
            tag[s] = None
            free.append(s)
            computing = False
        else:
            computing = False
        max_busy = max(max_busy, sum(1 for x in state if x != "Free"))
        try_issue_fetch()
        try_compute()
    completed = ci >= len(order) and nf >= len(fetches)
    return ReplayResult(completed, assignments, max_busy, ok_trans, ok_tags)


# --------------------------------------------------------------------------
# C-S7 stagger (derived; timing only).  Rank r starts its fetch stream at tick
# t_r = (-r) mod (d-1).  Realises PAPER.md:201 (ii) "different ranks tend to
# prefetch different layers" with S = 2 instead of d-1.
# --------------------------------------------------------------------------
def stagger_ticks(d: int, r: int) -> int:
    if d < 3:
        return 0
    return (-r) % (d - 1)


def owners_read_at_tick(owner: list[int], d: int, k: int, plans: list[list[int]],
                        offsets: list[int]) -> list:
    """Owner each rank is reading at global tick k (None before its start);
    each rank fetches plan entries back to back, one per tick, across passes."""
    out = []
    for r in range(d):
        j = k - offsets[r]
        if j < 0 or not plans[r]:
            out.append(None)
        else:
            out.append(owner[plans[r][j % len(plans[r])]])
    return out


def single_reader_violations(owner: list[int], d: int, ticks: int, plans, offsets) -> int:
    """Count ticks (after every rank started) at which two ranks read the same owner."""
    start = max(offsets) if offsets else 0
    bad = 0
    for k in range(start, start + ticks):
        cur = [o for o in owners_read_at_tick(owner, d, k, plans, offsets) if o is not None]
        if len(cur) != len(set(cur)):
            bad += 1
    return bad
