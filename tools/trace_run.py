"""One C3 sub-batch with the encoder's per-tile event trace (LOCC_TC_TRACE=1): prints the raw trace
(stderr of the library) for tools/trace_summary.py."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import locc_synth as ls  # noqa: E402
from paper_2304_09439_b200 import build  # noqa: E402

from paper_2304_09439_b200 import locc  # noqa: E402

# the trace is compiled in only in a diagnostic build (kernels_encoder_tc.cu LOCC_TRACE_BUILD)
locc.LIB_PATH = build.build(out="/tmp/liblocc_trace.so", flags=("-DLOCC_TRACE_BUILD=1",))

wl = ls.make_workload("C3", N=262144)
with locc.Locc(precision=locc.LOCC_PREC_BF16, device=0) as ctx:
    ctx.load_weights_mem(ls.weight_set("spread"))
    ctx.set_shapes(wl.points)
    ctx.query(wl.pairs[:65536], wl.poses[:65536])
    os.environ["LOCC_TC_TRACE"] = "1"
    ctx.query(wl.pairs, wl.poses)
