"""Strategy selection from measured cost curves.

Loads the config-2 sweep (h1 / h2 samples per compressor, tools/sweep.py),
builds the candidate GPU options of a tensor and picks, per tensor size, the
option with the smallest predicted sync time through the C ABI
(esp_select_option: the cost table, with h1/h2 fitted log-log, P:27;
Algorithm 1's GetBestOption, with no computation to overlap,
reading R21).  Host-side planning only: nothing here runs on the sync path.
"""
import json
import os

from . import esp as E

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEFAULT_SWEEP = os.path.join(ROOT, "profiles", "r01_sweep.json")

# candidate options: (kind, ratio, routine, process, sweep curve name)
CANDIDATES = [
    ("none", 1.0, "allreduce", 0, None),
    ("dgc", 0.01, "allgather", 0, "dgc_0.01"),
    ("dgc", 0.01, "alltoall_allgather", 1, "dgc_0.01"),
    ("dgc", 0.01, "alltoall_allgather", 2, "dgc_0.01"),
    ("dgc", 0.01, "gather_broadcast", 1, "dgc_0.01"),
    ("dgc", 0.01, "gather_broadcast", 2, "dgc_0.01"),
    ("randomk", 0.01, "allreduce", 0, "randomk_0.01"),
    ("randomk", 0.01, "allgather", 0, "randomk_0.01"),
    ("efsignsgd", 1.0, "allgather", 0, "efsignsgd_1.0"),
    ("efsignsgd", 1.0, "alltoall_allgather", 2, "efsignsgd_1.0"),
    ("efsignsgd", 1.0, "alltoall_allgather", 1, "efsignsgd_1.0"),
    ("efsignsgd", 1.0, "gather_broadcast", 2, "efsignsgd_1.0"),
    ("onebit", 1.0, "alltoall_allgather", 2, "onebit_1.0"),
]


def load_curves(path=DEFAULT_SWEEP):
    """{(compressor, op): [(input bytes, seconds), ...]} from a sweep JSON."""
    d = json.loads(open(path).read().strip().splitlines()[-1])
    return {(c["compressor"], c["op"]): [(s["size_bytes"], s["ns"] * 1e-9) for s in c["samples"]]
            for c in d["curves"]}


def marginal(samples, pieces=1):
    """B200 "bucketed" reading of a per-call curve: libesp launches once per
    bucket, so a tensor costs the curve minus its per-call floor (the first,
    smallest sample); `pieces` divides a fused multi-piece h2 curve into a
    per-piece cost so that the table's n h2 terms add up to one fused pass."""
    floor = samples[0][1]
    return [(b, max((t - floor) / pieces, 1e-9)) for b, t in samples]


def options(curves, candidates=CANDIDATES, model="paper"):
    """model = "paper": the per-call curves as measured (one kernel chain per
    tensor and one h2 per piece, as the cost table assumes); "bucketed": the
    per-tensor marginal cost with the 8-piece fused h2 curve (libesp's
    execution: one launch chain per bucket, n pieces decoded in one pass)."""
    out = []
    for kind, ratio, routine, proc, name in candidates:
        if name is None:
            out.append(E.make_option(kind, ratio, routine))
        elif model == "paper":
            out.append(E.make_option(kind, ratio, routine, h1=curves[(name, "h1")],
                                     h2=curves[(name, "h2_npieces1")], process=proc))
        else:
            out.append(E.make_option(kind, ratio, routine, h1=marginal(curves[(name, "h1")]),
                                     h2=marginal(curves[(name, "h2_npieces8")], 8), process=proc))
    return out


def candidates_for(algorithm=None):
    """"Given a DDL training job and a GC algorithm": the options are
    no compression plus every GPU option of that algorithm; None = all
    algorithms' options (a wider search than the paper's)."""
    if algorithm is None:
        return CANDIDATES
    return [c for c in CANDIDATES if c[0] in ("none", algorithm)]


class Selector:
    """Per-size choice for n ranks at B bytes/s; memoised."""

    def __init__(self, n, B=7.7e11, sweep=DEFAULT_SWEEP, candidates=None, model="paper", algorithm="dgc"):
        candidates = candidates if candidates is not None else candidates_for(algorithm)
        self.n, self.B, self.candidates = n, B, candidates
        self.opts = options(load_curves(sweep), candidates, model)
        self.memo = {}

    def choose(self, numel):
        """-> (index into candidates, predicted seconds)."""
        if numel not in self.memo:
            self.memo[numel] = E.select_option(self.opts, numel, self.n, self.B)
        return self.memo[numel]

    def rule(self, numel):
        """bench.py-style rule: numel -> (kind, ratio, routine, {process})."""
        kind, ratio, routine, proc, _ = self.candidates[self.choose(numel)[0]]
        return (kind, ratio, routine, {"process": proc}) if proc else (kind, ratio, routine)

    def predicted(self, idx, numel):
        return E.option_time(self.opts[idx], numel, self.n, self.B)
