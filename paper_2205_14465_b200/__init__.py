"""B200-native Espresso (arXiv 2205.14465) compressed gradient-sync hot path.

The product is libesp.so (CUDA kernels for sm_100a + NCCL, C ABI in
include/esp.h); `esp` is its ctypes binding.
"""
from . import esp  # noqa: F401
from .esp import (Ctx, World, esp_compress, esp_decompress, esp_sync, esp_sync_many,  # noqa: F401
                  esp_compressed_bytes, esp_wire_bytes, esp_model_time, esp_launch_count)
