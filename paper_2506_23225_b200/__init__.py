"""paper_2506_23225_b200 -- B200-native FlashMGLU forward (MoEG / SwiMGLU up-projection).

The product is ``libmglu.so`` (C ABI in ``include/mglu.h``, CUDA kernels for sm_100a in
``csrc/``).  ``mglu`` is its thin Python binding (marshalling only), ``shard`` the column-shard
launcher.  Nothing here imports the test oracle (``oracle/``).
"""
__all__ = ["mglu", "shard", "build"]


def __getattr__(name):
    if name in __all__:
        import importlib
        return importlib.import_module(f"{__name__}.{name}")
    raise AttributeError(name)
