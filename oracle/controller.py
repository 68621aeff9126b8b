"""Remapping Controller (oracle). TEST INFRASTRUCTURE ONLY.

Algorithm 1 and §5.1-5.2, written out over the
oracle allocator (c2), with the readings of DESIGN.md (NEXT-1):

  step (Alg. 1 line 3): if the active model cannot get its blocks,
      remapping() and retry, until it fits or nothing is left to remap;
  remapping() (lines 14-23): victim = the inactive model with the lowest
      priority (unset = 0); ties -> the most recently activated (MRU);
      models that reached cap * layers are skipped (Alg. 1 line 20 drops a
      model at remapped == layers). Reclaim its highest remaining layers,
      layers_per_call at a time, beta = 0, into the active model;
  Dynamic Reversion (lines 7-12): regions of the active
      model, newest first, whose blocks are all free are given back while at
      least `headroom` blocks stay free; a region with at most migrate_max live
      blocks is emptied first by moving them out (reading #29);
  activation: the newly active model's donated regions are reverted first.

Pinned by the directional checks in tests/test_controller_cpu.py (victim order
under priorities and MRU, cap, LIFO reversion) and by parity of its action log
with the product controller on seeded traces.
"""
from .allocator import NoBlocks


class Controller:
    def __init__(self, alloc, models, active, cap=1.0, layers_per_call=1, order="mru"):
        self.al = alloc
        self.n = {m: v[0] for m, v in models.items()}
        self.prio = {m: (v[1] if v[1] is not None else 0) for m, v in models.items()}
        self.taken = {m: set() for m in models}
        self.last_act = {m: 0 for m in models}
        self.cap, self.k = cap, layers_per_call
        self.sign = -1 if order == "mru" else 1   # MRU: most recently activated first
        self.t = 0
        self.log = []
        self.active = None
        self.activate(active)

    def limit(self, m):
        return int(self.cap * self.n[m] + 1e-9)

    def remapping(self):
        best = None
        for m in sorted(self.n):
            if m == self.active or len(self.taken[m]) >= self.limit(m):
                continue
            if len(self.taken[m]) + len(self.al.models[m].cycle) >= self.n[m]:
                continue
            key = (self.prio[m], self.sign * self.last_act[m], m)
            if best is None or key < best[0]:
                best = (key, m)
        if best is None:
            return None
        m = best[1]
        own = set(self.al.models[m].cycle)       # its own streaming cycle is not donatable
        remaining = [l for l in range(self.n[m] - 1, -1, -1) if l not in self.taken[m] and l not in own]
        layers = sorted(remaining[: min(self.k, self.limit(m) - len(self.taken[m]))])
        gained = self.al.remap(m, self.active, layers, 0)
        self.taken[m] |= set(layers)
        entry = ("remap", m, tuple(layers), gained)
        self.log.append(entry)
        return entry

    def alloc(self, seq, n):
        while True:
            try:
                return self.al.alloc(self.active, seq, n)
            except NoBlocks:
                if self.remapping() is None:
                    raise

    def free(self, seq):
        self.al.free_seq(self.active, seq)

    def revert(self, headroom, migrate_max=0):
        """Dynamic Reversion, newest region first. A region still holding at most
        migrate_max live blocks is first emptied by migrate (reading #29)."""
        out = []
        regs = self.al.models[self.active].regions
        for idx in reversed(range(len(regs))):
            g = regs[idx]
            if g["retired"]:
                continue
            # the regions of a streaming cycle revert as one (allocator.unremap)
            ids = self.al._region_ids(self.al.models[self.active], idx)
            live = sum(1 for i in ids if i not in self.al.models[self.active].free)
            if live > migrate_max:
                continue
            if len(self.al.models[self.active].free) - len(ids) < headroom:
                continue
            n_layers = (sum(r["n_layers"] for r in regs if r["cycle"] and r["donor"] == g["donor"] and not r["retired"])
                        if g["cycle"] else g["n_layers"])
            if live:
                moves = self.al.migrate(self.active, idx)
                self.log.append(("migrate", idx, len(moves)))
                out.append(self.log[-1])
            self.al.unremap(self.active, idx)
            self.taken[g["donor"]] -= set(range(g["first_layer"], g["first_layer"] + g["n_layers"]))
            entry = ("revert", idx, g["donor"], n_layers)
            self.log.append(entry)
            out.append(entry)
        return out

    def activate(self, model):
        self.t += 1
        if self.active is not None and self.active != model:
            for owner in sorted(self.n):
                if owner == model:
                    continue
                for idx, g in enumerate(self.al.models[owner].regions):
                    if g["donor"] == model and not g["retired"]:
                        self.al.unremap(owner, idx)
                        self.log.append(("revert", idx, model, g["n_layers"]))
            self.taken[model] = set()
            self.al.set_active(self.active, False)
        for m in self.n:
            if m != model:
                self.al.set_active(m, False)
        self.al.set_active(model, True)
        self.last_act[model] = self.t
        self.active = model
        self.log.append(("activate", model))
