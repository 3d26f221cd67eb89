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
    ("dgc", 0.01, "gather_broadcast", 2, "dgc_0.01"),
    ("randomk", 0.01, "allreduce", 0, "randomk_0.01"),
    ("randomk", 0.01, "allgather", 0, "randomk_0.01"),
    ("efsignsgd", 1.0, "allgather", 0, "efsignsgd_1.0"),
    ("efsignsgd", 1.0, "alltoall_allgather", 2, "efsignsgd_1.0"),
    ("efsignsgd", 1.0, "gather_broadcast", 2, "efsignsgd_1.0"),
    ("onebit", 1.0, "alltoall_allgather", 2, "onebit_1.0"),
]


def load_curves(path=DEFAULT_SWEEP):
    """{(compressor, op): [(input bytes, seconds), ...]} from a sweep JSON."""
    d = json.loads(open(path).read().strip().splitlines()[-1])
    return {(c["compressor"], c["op"]): [(s["size_bytes"], s["ns"] * 1e-9) for s in c["samples"]]
            for c in d["curves"]}


def options(curves, candidates=CANDIDATES, h2_op="h2_npieces1"):
    out = []
    for kind, ratio, routine, proc, name in candidates:
        if name is None:
            out.append(E.make_option(kind, ratio, routine))
        else:
            out.append(E.make_option(kind, ratio, routine, h1=curves[(name, "h1")], h2=curves[(name, h2_op)],
                                     process=proc))
    return out


class Selector:
    """Per-size choice for n ranks at B bytes/s; memoised."""

    def __init__(self, n, B=7.7e11, sweep=DEFAULT_SWEEP, candidates=CANDIDATES):
        self.n, self.B, self.candidates = n, B, candidates
        self.opts = options(load_curves(sweep), candidates)
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
