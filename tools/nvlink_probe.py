"""Which NVML NVLink byte counters move on this box?  Copies 1 GiB from GPU 0
to GPU 1 with torch (peer copy over NVLink) and prints every candidate
counter's return code and delta (diagnostic for bench.py's link fields)."""
import pynvml as nv
import torch

nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(0)
F = {"THROUGHPUT_DATA_TX": nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX,
     "THROUGHPUT_DATA_RX": nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX,
     "THROUGHPUT_RAW_TX": nv.NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX,
     "THROUGHPUT_RAW_RX": nv.NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_RX}


def read():
    out = {}
    for name, fid in F.items():
        for scope in (0, 0xFFFFFFFF):
            try:
                v = nv.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
                out[(name, scope)] = (v.nvmlReturn, int(v.value.ullVal))
            except Exception as e:  # noqa: BLE001
                out[(name, scope)] = (repr(e), 0)
    for link in range(18):
        for name, fid in (("XMIT_BYTES", nv.NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES),
                          ("RCV_BYTES", nv.NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES)):
            try:
                v = nv.nvmlDeviceGetFieldValues(h, [(fid, link)])[0]
                out[(name, link)] = (v.nvmlReturn, int(v.value.ullVal))
            except Exception as e:  # noqa: BLE001
                out[(name, link)] = (repr(e), 0)
    try:
        for link in range(2):
            out[("util_counter0", link)] = (0, nv.nvmlDeviceGetNvLinkUtilizationCounter(h, link, 0)[0])
    except Exception as e:  # noqa: BLE001
        out[("util_counter0", 0)] = (repr(e), 0)
    return out


a = torch.empty(1 << 28, dtype=torch.float32, device="cuda:0")
b = torch.empty(1 << 28, dtype=torch.float32, device="cuda:1")
b.copy_(a)
torch.cuda.synchronize(0)
torch.cuda.synchronize(1)
r0 = read()
for _ in range(4):
    b.copy_(a)
torch.cuda.synchronize(0)
torch.cuda.synchronize(1)
r1 = read()
print("4 GiB GPU0 -> GPU1")
for k in r0:
    print(k, "ret", r0[k][0], r1[k][0], "delta", r1[k][1] - r0[k][1])
