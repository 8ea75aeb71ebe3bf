"""CPU oracle for the FlashMGLU forward pass -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything from this package.  The product package
``paper_2506_23225_b200`` never imports it, and the two share no code (no kernels, headers,
helpers, tables or constants).  Inputs reach both sides only through ``synth/`` (seeded
generators holding none of the method's arithmetic).

Contents
  * ``mglu_ref``    -- numpy float64 twin: Eq. 3 written with explicit masked matrices.
  * ``mglu_oracle.c`` (+ ``c_oracle``) -- plain C, binary64 loops, OpenMP over output columns.
  * ``accounting``  -- closed forms of Table 1 / Sec. 4.1 (memory load, parameters, FLOPs).
  * ``codes``       -- per-element mask code streams.
  * ``backward``    -- the training path: Eq. 3's gradients under Alg. 2's STE.

Every function cites the PAPER.md passage it follows (``P:<line>``).  DESIGN.md lists the
readings (R1..R15) taken where the paper is silent or garbled.

Parity pins: every function here is pinned by ``tests/test_oracle_pins.py`` against values the
paper prints, closed forms, exact rational brute force and special cases -- see that file.
"""
from .mglu_ref import (  # noqa: F401
    ACT_IDENTITY, ACT_SWISH, ACT_GELU, ACT_RELU, ACT_SIGMOID, ACT_NAMES,
    act_np, decode_bf16, pack_np, unpack_np, mglu_forward_np, mglu_partials_np,
)
from . import accounting  # noqa: F401
from .c_oracle import COracle, build_c_oracle  # noqa: F401
from .topk import router_logits, topk_gate, mglu_routed_from_partials  # noqa: F401,E402
from .ffn import ffn_forward_np, dense_np  # noqa: F401,E402
from .variants import VARIANTS, mglu_variant_from_streams  # noqa: F401,E402
from .codes import codes_to_bits_np, bits_to_codes_np  # noqa: F401,E402
from .backward import act_grad_np, mglu_backward_np, relaxed_forward_np  # noqa: F401,E402
