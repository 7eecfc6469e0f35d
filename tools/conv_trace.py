"""Dev tool: per-CTA timeline of each conv launch of the bench step (libsphinx_trace.so).

    python -m paper_2511_18672_b200.build --trace && python tools/conv_trace.py

For conv launch j of a warm step, the trace build records per CTA (globaltimer, ns): entry,
after pdl_wait, first MMA, last MMA commit, epilogue done, exit, chunks issued.  Printed relative
to the earliest entry: launch skew, prologue, fill, main loop vs the ideal, drain and tail.
"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_18672_b200 as sp  # noqa: E402

lib = sp.load(os.path.join(ROOT, "paper_2511_18672_b200", "libsphinx_trace.so"))
import bench  # noqa: E402
import torch  # noqa: E402

dev = torch.device("cuda", 0)
st = bench.GpuStep(bench.make_request("r0"), dev)
n_conv = 3 * bench.CONVS_PER_LEVEL
for _ in range(3):
    st.run()
torch.cuda.synchronize()
base = 3 * n_conv
sms = torch.cuda.get_device_properties(0).multi_processor_count
buf = (ctypes.c_ulonglong * (sms * 24))()
zero = (ctypes.c_ulonglong * (sms * 24))()
for j in range(n_conv):
    lib.sphinx_debug_conv_trace_reset()
    os.environ["SPHINX_TRACE_LAUNCH"] = str(base + j)
    st.run()
    torch.cuda.synchronize()
    base += n_conv
    assert lib.sphinx_debug_conv_trace(buf, sms) == 0
    a = np.frombuffer(buf, dtype=np.uint64).reshape(sms, 24).astype(np.int64)
    live = a[:, 0] > 0
    a = a[live]
    t0 = a[:, 0].min()
    rel = lambda c: (a[:, c] - t0) / 1e3  # us
    lead = a[:, 2] > 0
    chunks = a[lead, 6]
    print(f"conv {j} (level {j // bench.CONVS_PER_LEVEL}): {live.sum()} CTAs, "
          f"kernel span {(a[:, 5].max() - t0) / 1e3:.1f} us")
    for name, c in (("entry", 0), ("after pdl_wait", 1), ("setup done", 15), ("first A issued", 8), ("first B issued", 9),
                    ("first A full", 10), ("first MMA", 2), ("last MMA", 3), ("last acc ready", 11),
                    ("epilogue done", 4), ("exit", 5), ("B producer done", 7),
                    ("split parked", 16), ("split rendezvous", 17), ("split reduced", 18)):
        v = rel(c)[a[:, c] > 0]
        if len(v):
            print(f"   {name:16s} min {v.min():7.2f}  med {np.median(v):7.2f}  max {v.max():7.2f}")
    sp_ = a[:, 16] > 0
    if sp_.any():
        print(f"   split units: {sp_.sum()} CTAs, ns {np.unique(a[sp_, 19])}; last acc->parked med "
              f"{np.median((a[sp_, 16] - a[sp_, 11]) / 1e3):.2f} us, parked->rendezvous med "
              f"{np.median((a[sp_, 17] - a[sp_, 16]) / 1e3):.2f} us (max {np.max((a[sp_, 17] - a[sp_, 16]) / 1e3):.2f}), "
              f"reduce med {np.median((a[sp_, 18] - a[sp_, 17]) / 1e3):.2f} us")
    nt_ = np.maximum(a[:, 12], 1)
    print(f"   epilogue tiles med {np.median(a[:, 12]):.0f}; TMEM drain per tile med "
          f"{np.median(a[:, 13] / nt_) / 1e3:.2f} us, last tile med {np.median(a[:, 14]) / 1e3:.2f} us; "
          f"last acc -> epilogue done per CTA med {np.median((a[:, 4] - a[:, 11]) / 1e3):.2f} us")
    mm = (a[lead, 3] - a[lead, 2]) / 1e3
    print(f"   main loop per leader: med {np.median(mm):.2f} us, chunks med {np.median(chunks):.0f} "
          f"(min {chunks.min()}, max {chunks.max()}), us/chunk med {np.median(mm / np.maximum(chunks, 1)):.3f}")
