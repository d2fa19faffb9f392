"""Debug-only: build libds2ctc with -DDS2CTC_EPOCH_TIMING and print per-epoch
warp busy cycles of the first cluster for one workload (design evidence)."""
import ctypes
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
CSRC = os.path.join(ROOT, "paper_1512_02595_b200", "csrc")
OUT = os.path.join(ROOT, "build", "epoch_timing")


def build(defines=()):
    os.makedirs(OUT, exist_ok=True)
    tag = "_".join(d.lower() for d in defines) or "base"
    so = os.path.join(OUT, f"libds2ctc_timing_{tag}.so")
    srcs = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    if os.path.exists(so) and all(os.path.getmtime(f) <= os.path.getmtime(so) for f in srcs):
        return so  # prebuilt (e.g. shipped with the snapshot)
    objs = []
    from concurrent.futures import ThreadPoolExecutor

    from paper_1512_02595_b200.build import CU_FLAGS, CU_SOURCES

    def cc(src):
        obj = os.path.join(OUT, tag + src + ".o")
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-lineinfo",
                        *CU_FLAGS.get(src, []), "-DDS2CTC_EPOCH_TIMING", *[f"-DDS2CTC_EXP_{d}" for d in defines],
                        "-Xcompiler", "-fPIC", f"-I{ROOT}/include", f"-I{CSRC}", "-c",
                        os.path.join(CSRC, src), "-o", obj], check=True)
        return obj

    with ThreadPoolExecutor(len(CU_SOURCES)) as ex:
        objs.extend(ex.map(cc, CU_SOURCES))
    for src in ("ctc_api.cpp", "scheduler.cpp"):
        obj = os.path.join(OUT, src + ".o")
        subprocess.run(["g++", "-O2", "-std=c++17", "-fPIC", f"-I{ROOT}/include", f"-I{CSRC}",
                        "-I/usr/local/cuda/include", "-c", os.path.join(CSRC, src), "-o", obj], check=True)
        objs.append(obj)
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static", "-o", so,
                    *objs], check=True)
    return so


def run(so, A=29, T=700, L=150, B=64, brief=False):
    import torch

    from paper_1512_02595_b200 import _lib
    from paper_1512_02595_b200.synth import fixed_shape_batch

    os.environ["DS2CTC_LIB"] = so  # variant: tolerate entry points an older build lacks
    _lib.LIB_PATH = so
    _lib._lib = None
    from paper_1512_02595_b200 import ctc

    acts, flat, ll, il = fixed_shape_batch(A, T, L, B)
    x = torch.from_numpy(acts).cuda()
    for _ in range(3):
        ctc.compute_ctc_loss(x, flat, ll, il)
    torch.cuda.synchronize()
    buf = np.zeros((2, 128, 33, 2), dtype=np.int64)
    lib = ctypes.CDLL(so)
    assert lib.ds2ctc_debug_epoch_clocks(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong))) == 0
    steps = np.zeros((2, 8, 32, 4), dtype=np.int64)
    assert lib.ds2ctc_debug_step_clocks(steps.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong))) == 0
    for cta in range(2):
        base = steps[cta, 0, 0, 0]
        print(f"CTA {cta} epoch-1 step stamps (relative to warp 0 step 0 start): [start, mid, end] per warp")
        for k in range(0, 32, 4):
            row = []
            for w in range(8):
                if steps[cta, w, k, 0] == 0:
                    continue
                row.append(f"w{w}:" + ",".join(str(int(steps[cta, w, k, j] - base)) for j in range(3)))
            print(f"  k+{k:2d} " + "  ".join(row))
    print("TIGHT cycles/step: critical", steps[0, 7, 31, 3] / 1000.0, "| + load_emis", steps[0, 7, 31, 2] / 1000.0,
          "| + stamps & real k", steps[0, 7, 31, 1] / 1000.0)
    meetbuf = np.zeros(18, dtype=np.int64)
    if lib.ds2ctc_debug_meet_clocks(meetbuf.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong))) == 0:
        meet = meetbuf[:16].reshape(2, 8)
        for cta in range(2):
            m = meet[cta]
            e0 = buf[cta, 0, 0, 0]
            last = max(int(buf[cta, e, w, 1]) for e in range(128) for w in range(33) if buf[cta, e, w, 1] > 0)
            print(f"  cta{cta}: kernel: prologue {e0 - m[6]}, epochs {last - e0}, after-epochs {m[7] - last}, "
                  f"tail {meetbuf[16 + cta] - m[7]}, total {meetbuf[16 + cta] - m[6]}")
            print(f"  cta{cta}: meet: store+wait {m[1]-m[0]}, cluster barrier {m[2]-m[1]}, logZ {m[3]-m[2]}, "
                  f"shift+load {m[4]-m[3]}, sync {m[5]-m[4]}")
    pro = np.zeros((2, 8, 8), dtype=np.int64)
    if hasattr(lib, "ds2ctc_debug_prologue_clocks") and \
            lib.ds2ctc_debug_prologue_clocks(pro.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong))) == 0:
        meetbuf2 = np.zeros(18, dtype=np.int64)
        lib.ds2ctc_debug_meet_clocks(meetbuf2.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)))
        for cta in range(2):
            start = meetbuf2[cta * 8 + 6]
            rows = []
            for pt in range(5):
                v = [int(pro[cta, pt, w] - start) if pro[cta, pt, w] else None for w in range(6)]
                rows.append(f"p{pt}:" + ",".join("-" if x is None else str(x) for x in v))
            print(f"  cta{cta}: prologue stamps (per warp 0..5, from kernel start) " + "  ".join(rows))
    if brief:
        for cta in range(2):
            rows = [buf[cta, e] for e in range(128) if buf[cta, e, 0, 0] != 0]
            p1 = [r for r in rows[:8]]
            p2 = [r for r in rows[-8:-1]]
            busy2 = np.mean([[int(r[w, 1] - r[w, 0]) for w in range(8)] for r in p2], axis=0)
            print(f"  cta{cta}: phase-2 epoch busy per warp {busy2.astype(int).tolist()}")
            sv = steps[cta, 7]
            for ep in (2, len(rows) - 3):
                if 0 < ep < 32 and sv[ep, 0] > 0:
                    print(f"  cta{cta}: service epoch {ep}: stage {sv[ep,1]-sv[ep,0]}, wait {sv[ep,2]-sv[ep,1]}, "
                          f"convert {sv[ep,3]-sv[ep,2]}, grad_write {steps[cta, 6, ep, 0] - sv[ep,3]}")
            busy = np.mean([[int(r[w, 1] - r[w, 0]) for w in range(8)] for r in p1], axis=0)
            # service = warp 0, chain warps 1..NCW; per-step cycles over the stamped phase-2 epoch
            for w in (1, 2, 3):
                st = steps[cta, w]
                n = int((st[:, 0] > 0).sum())
                if n > 1:
                    per = (st[n - 1, 0] - st[0, 0]) / (n - 1)
                    print(f"  cta{cta}: chain warp {w} phase-2 cycles/step {per:.0f}, "
                          f"step body {np.mean(st[1:n, 2] - st[1:n, 0]):.0f}")
            total = int(rows[-1][0, 1] - rows[0][0, 0])
            print(f"  cta{cta}: total {total} cycles, phase-1 epoch busy per warp {busy.astype(int).tolist()}")
        return
    for cta in range(2):
        e0 = buf[cta, 0, 0, 0]
        print(f"CTA {cta} ({'fwd' if cta == 0 else 'bwd'})")
        for e in range(128):
            row = buf[cta, e]
            if row[0, 0] == 0:
                break
            busy = [int(row[w, 1] - row[w, 0]) for w in range(33) if row[w, 0] > 0]
            start = int(row[0, 0] - e0)
            print(f"  epoch {e:3d} start {start:8d}  busy per warp {busy}")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "variants":
        sets = [tuple(v.split("+")) if v != "base" else () for v in sys.argv[2:]] or [()]
        shape = [int(v) for v in os.environ.get("SHAPE", "29,700,150,64").split(",")]  # A,T,L,B
        for defs in sets:
            so = build(defs)
            print("variant", defs or "base", "shape", shape)
            run(so, *shape, brief=True)
    else:
        so = build()
        args = [int(v) for v in sys.argv[1:]]
        run(so, *args)
