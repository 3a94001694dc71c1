"""B200-native sparse-causal chunk attention (TalkingMachines, arXiv 2506.03099).

The product is libtm.so (include/tm.h); `paper_2506_03099_b200.tm` is its thin
ctypes binding.  The binding is loaded on first use (so `python -m
paper_2506_03099_b200.build` can rebuild a stale library); using it without a
built libtm.so raises ImportError -- there is no CPU fallback.
"""
_EXPORTS = ("TM_BF16", "TM_FP32", "ChunkAttention", "TMError", "make_config",
            "tm_flow_euler_step")


def __getattr__(name):
    if name == "tm" or name in _EXPORTS:
        import importlib
        tm = importlib.import_module(".tm", __name__)
        return tm if name == "tm" else getattr(tm, name)
    raise AttributeError(name)
