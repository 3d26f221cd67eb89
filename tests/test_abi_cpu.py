"""C-ABI checks that need no GPU: the library loads, exports every symbol
include/esp.h declares, and its host-side size / cost-table functions agree
with the oracle's independent implementations."""
import re
import os

import pytest

from oracle import esp_oracle as O


@pytest.fixture(scope="module")
def E():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2205_14465_b200 import esp
    return esp


def test_exports_every_declared_symbol(E):
    hdr = open(os.path.join(os.path.dirname(__file__), "..", "include", "esp.h")).read()
    declared = set(re.findall(r"\b(esp_[a-z0-9_]+)\s*\(", hdr))
    assert declared == set(E.SYMBOLS)
    L = E.lib()
    for s in declared:
        assert hasattr(L, s), s
    assert E.lib().esp_status_string(2) == b"ESP_ERR_UNSUPPORTED"


@pytest.mark.parametrize("kind", ["dgc", "topk", "randomk", "efsignsgd", "onebit", "none"])
def test_compressed_bytes_vs_oracle(E, kind):
    for N in (1, 31, 32, 33, 1000, 4097, 2 ** 20, 10 ** 6, 31_254_528):
        for P in (1, 2, 4, 8):
            for ratio in (0.001, 0.01, 1.0):
                got = E.esp_compressed_bytes(E.cfg_of(kind, ratio), N, P)
                assert got == O.chunk_bytes(O.Cfg(kind, ratio), N, P) * P, (N, P, ratio)


def test_too_large(E):
    with pytest.raises(E.EspError) as ei:
        E.esp_compressed_bytes(E.cfg_of("dgc"), 1 << 31, 1)
    assert ei.value.status == 3


def test_wire_bytes_vs_oracle(E):
    rows = {("allreduce", "allreducible"): "allreduce", ("allgather", "sparse"): "allgather",
            ("allgather", "quantized"): "allgather",
            ("alltoall_allgather", "sparse"): "alltoall_allgather_sparse",
            ("alltoall_allgather", "quantized"): "alltoall_allgather_quantized",
            ("gather_broadcast", "sparse"): "gather_broadcast_sparse",
            ("gather_broadcast", "quantized"): "gather_broadcast_quantized"}
    for (routine, tt), row in rows.items():
        for n in (1, 2, 4, 8):
            for M in (2 ** 16, 2 ** 20, 2 ** 24, 1e8):
                sent, recv = E.esp_wire_bytes(routine, tt, M, n)
                assert recv == pytest.approx(O.table_comm_bytes(row, M, n)) and sent == recv
    # S:132 worked example through the library; S:126 for the uncompressed pairs
    assert E.esp_model_time("allreduce", "allreducible", 1e8, 4, 1.25e10) == pytest.approx(0.012)
    assert E.esp_model_time("reducescatter_allgather", "allreducible", 1e8, 4, 1.25e10) == pytest.approx(0.012)
    assert E.esp_model_time("reduce_broadcast", "allreducible", 1e8, 4, 1.25e10) == pytest.approx(0.032)
    for routine, tt in (("allreduce", "sparse"), ("allgather", "allreducible"), ("reduce_broadcast", "quantized")):
        with pytest.raises(E.EspError) as ei:
            E.esp_wire_bytes(routine, tt, 1e6, 4)
        assert ei.value.status == 2
