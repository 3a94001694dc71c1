"""Helpers for GPU parity tests: move synthetic inputs to torch CUDA tensors
(bit-identical to what the oracle reads) and compare against the oracle."""
import numpy as np
import torch

from synthetic import inputs as syn

BF16_TOL = 2e-2      # BJ.north_star: max|err| <= 2e-2 * max|O| (bf16 I/O, fp32 accumulate)
BF16_ALARM = 8e-3    # internal alarm (emulated kernel error ~3e-3)
FP32_TOL = 1e-4      # BJ.north_star fp32 validation mode


def to_dev(t: syn.Tensor, device="cuda"):
    if t.dtype == "bf16":
        x = torch.from_numpy(t.store.view(np.int16)).to(device)
        return x.view(torch.bfloat16)
    return torch.from_numpy(t.store).to(device)


def from_dev(x: torch.Tensor) -> np.ndarray:
    """Device tensor -> fp64 numpy (exact upcast)."""
    if x.dtype == torch.bfloat16:
        return syn.bf16_bits_to_f64(x.view(torch.int16).cpu().numpy().view(np.uint16))
    return x.double().cpu().numpy()


def rel_err(o, ref):
    o = np.asarray(o, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert np.isfinite(o).all(), "non-finite output"
    return float(np.abs(o - ref).max() / np.abs(ref).max())


def sample_rows(L, k=61, seed=0):
    rng = np.random.default_rng(seed)
    rows = set([0, 1, L - 1, L - 2, 127, 128, min(255, L - 1)])
    rows |= set(int(x) for x in rng.choice(L, size=min(k, L), replace=False))
    return np.array(sorted(r for r in rows if 0 <= r < L), dtype=np.int64)


_cudart = None


def dev_copy(dst_ptr: int, src_ptr: int, nbytes: int) -> None:
    """Synchronous device-to-device copy between raw pointers (test plumbing)."""
    global _cudart
    import ctypes
    if _cudart is None:
        _cudart = ctypes.CDLL("libcudart.so.12")
        _cudart.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                       ctypes.c_int]
    torch.cuda.synchronize()
    r = _cudart.cudaMemcpy(dst_ptr, src_ptr, nbytes, 3)   # cudaMemcpyDeviceToDevice
    torch.cuda.synchronize()
    assert r == 0, f"cudaMemcpy failed: {r}"
