"""B200-native NQKV hot path (arXiv 2505.16210): NF4 KV-cache quantize/append
and fused dequant-in-registers decode attention, exposed through the C ABI in
include/nqkv.h (libnqkv.so) and the thin binding in .nqkv."""
__all__ = ["nqkv", "build"]
