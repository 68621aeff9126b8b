"""Remapping Controller (§5, Algorithm 1; SURVEY.md
NEXT-1) driving libmirage through the C-ABI.

Host-side policy, as in the paper (a Python component of the serving system):

* when the active model runs out of KV blocks, ``remapping()`` reclaims one more
  layer of the lowest-priority inactive model (Alg. 1 lines 14-23; P:373-388
  "prioritizes remapping parameters from inactive models with the lowest
  priority"; without priorities, round robin with Most-Recently-Used first,
  P:380-383), up to a per-model cap of the model's layers (P:387 threshold;
  Alg. 1 P:530 removes a model at remapped == layers, reading #8);
* when KV usage subsides, Dynamic Reversion gives empty reclaimed regions back
  to parameters, newest first (Alg. 1 lines 7-12), keeping
  ``headroom`` free blocks;
* activating an inactive model first reverts the regions it donated (its
  parameters must be resident to run).

Layer choice for an inactive donor (unstated by the paper, reading in
DESIGN.md): highest remaining layer index first, ``layers_per_call`` at a time;
layers of the donor's own streaming cycle (if it self-remapped while active)
are never donated.

``cap`` defaults to 1.0, a deliberate reading (#8): P:387 enforces a maximum
remapping threshold so enough parameters stay resident for a cold start, but
Alg. 1 removes a model only at remapped == layers and BASELINE C3 asks
for a fully remapped inactive tenant. The price of cap = 1.0 is the cold start:
every layer must be reloaded before (or, NEXT-4b, while) the tenant prefills.

Active-model self-remap (streaming), when no inactive model is left: with
``self_remap="auto"`` the controller applies §5.3: with T_T the
profiled per-layer transfer time (layer bytes / ``host_link_gbs``) and T_Compute
the measured decode time per token, it remaps alpha = 1 more layer only if
T_T * N <= T_Compute admits N >= 1 and the §5.4 planner finds a zero-stall
cycle (mirage_plan, BETA_DYNAMIC); otherwise it declines (logged). A callable
may be passed instead.
"""
from . import _lib


class RemappingController:
    def __init__(self, ctx, models, active, cap=1.0, layers_per_call=1, self_remap=None, host_link_gbs=None,
                 order="mru"):
        """models: {model_id: (n_layers, priority or None)}; active: model id;
        order: "mru" (the paper's default) or "lru" (the ablation)."""
        self.link_gbs = host_link_gbs
        self.order = order
        self.ctx = ctx
        self.info = {m: {"layers": n, "prio": p, "remapped": [], "act": 0} for m, (n, p) in models.items()}
        self.cap, self.per_call, self.self_remap = cap, layers_per_call, self_remap
        self.clock = 0
        self.log = []
        self.active = None
        self.activate(active)

    # ---- Metadata Store views ---------------------------------------------------
    def enable_remap(self):
        return any(not r["retired"] for r in self.ctx.regions(self.active))

    def _cycled(self, m):
        """Layers of m's own streaming cycle (slots and streamed layers): not donatable."""
        return set(self.ctx.query(m)["cycle"])

    def _candidates(self):
        out = []
        for m, i in self.info.items():
            if m == self.active:
                continue
            if len(i["remapped"]) >= int(self.cap * i["layers"] + 1e-9):
                continue
            if len(i["remapped"]) + len(self._cycled(m)) >= i["layers"]:
                continue
            prio = i["prio"] if i["prio"] is not None else 0
            rec = -i["act"] if self.order == "mru" else i["act"]
            out.append((prio, rec, m))            # lowest priority, then most (MRU) / least (LRU) recent
        return [m for _, _, m in sorted(out)]

    # ---- Alg. 1 remapping() -----------------------------------------------------
    def remapping(self):
        cands = self._candidates()
        if not cands:
            if self.self_remap == "auto":
                return self._auto_self_remap()
            if self.self_remap is not None:
                act = self.self_remap(self)
                if act:
                    self.log.append(("self_remap",) + tuple(act))
                return act
            return None
        m = cands[0]
        i = self.info[m]
        left = [l for l in range(i["layers"]) if l not in i["remapped"] and l not in self._cycled(m)]
        limit = int(self.cap * i["layers"] + 1e-9) - len(i["remapped"])
        take = sorted(left, reverse=True)[: min(self.per_call, limit)]
        layers = sorted(take)
        gained, _ = self.ctx.remap_layers(m, self.active, layers, 0)
        i["remapped"].extend(layers)
        act = ("remap", m, tuple(layers), gained)
        self.log.append(act)
        return act

    def _auto_self_remap(self):
        st = self.ctx.query(self.active)
        if st["m"] or not self.link_gbs or st["last_step_ms"] <= 0:
            return None
        n = self.info[self.active]["layers"]
        tt = int(st["layer_bytes"] / (self.link_gbs * 1e9) * 1e9)      # T_T, ns
        tcomp = int(st["last_step_ms"] * 1e6)                           # T_Compute per token, ns
        if tcomp // max(tt, 1) < 1:                                      # §5.3: T_T * N <= T_Compute
            self.log.append(("self_remap_declined", tt, tcomp))
            return None
        try:
            cycle, m, beta = _lib.plan(n, 1, _lib.BETA_DYNAMIC, tt, max(1, tcomp // n))
        except _lib.MirageError:
            self.log.append(("self_remap_declined", tt, tcomp))
            return None
        gained, _ = self.ctx.remap_layers(self.active, self.active, cycle, beta)
        act = ("self_remap", tuple(cycle), beta, gained)
        self.log.append(act)
        return act

    def alloc(self, seq, n):
        """alloc_blocks on the active model, remapping on shortfall (Alg. 1 line 3)."""
        while True:
            try:
                return self.ctx.alloc_blocks(self.active, seq, n)
            except _lib.MirageError as e:
                if e.code != _lib.ERR_NO_BLOCKS:
                    raise
                if self.remapping() is None:
                    raise

    def free(self, seq):
        self.ctx.free_blocks(self.active, seq)

    # ---- Dynamic Reversion ----------------------------------------------------------
    def revert(self, headroom, migrate_max=0):
        """Revert regions newest-first while free blocks stay >= headroom. A region
        still holding at most migrate_max live blocks is emptied first by
        mirage_migrate_region (reading #29)."""
        done = []
        regs = self.ctx.regions(self.active)
        for idx in range(len(regs) - 1, -1, -1):
            regs = self.ctx.regions(self.active)
            r = regs[idx]
            if r["retired"]:
                continue
            # a streaming cycle's regions revert (and migrate) together: count them all
            group = ([g for g in regs if g["cycle"] and g["donor"] == r["donor"] and not g["retired"]]
                     if r["cycle"] else [r])
            live = sum(g["n_blocks"] - g["n_free"] for g in group)
            n_blocks = sum(g["n_blocks"] for g in group)
            if live > migrate_max:
                continue
            free = self.ctx.query(self.active)["free_blocks"]
            if free - n_blocks < headroom:
                continue
            if live:
                moved = self.ctx.migrate_region(self.active, idx)
                self.log.append(("migrate", idx, moved))
                done.append(self.log[-1])
            self.ctx.unremap(self.active, idx)
            lay = set(range(r["first_layer"], r["first_layer"] + r["n_layers"]))
            if r["donor"] in self.info:
                i = self.info[r["donor"]]
                i["remapped"] = [l for l in i["remapped"] if l not in lay]
            act = ("revert", idx, r["donor"], sum(g["n_layers"] for g in group))
            self.log.append(act)
            done.append(act)
        return done

    # ---- temporal sharing -------------------------------------------------------------
    def activate(self, model):
        """Make `model` the active model; its donated regions are reverted first."""
        self.clock += 1
        if self.active is not None and self.active != model:
            # the model's parameters must be resident before it runs
            for owner in sorted(self.info):
                regs = self.ctx.regions(owner)
                for idx, r in enumerate(regs):
                    if r["donor"] == model and not r["retired"] and owner != model:
                        self.ctx.unremap(owner, idx)
                        self.log.append(("revert", idx, model, r["n_layers"]))
            self.info[model]["remapped"] = []
            self.ctx.set_active(self.active, False)
        for m in self.info:
            if m != model:
                self.ctx.set_active(m, False)
        self.ctx.set_active(model, True)
        self.info[model]["act"] = self.clock
        self.active = model
        self.log.append(("activate", model))
