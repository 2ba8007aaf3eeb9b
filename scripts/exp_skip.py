"""What-if: time the top C4 GEMM shape with A or B tile loads skipped
(TNB_EXP_SKIP; wrong results, timing only) to see how much the L2->SM
operand traffic costs under the power cap."""
import os, sys, subprocess, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1:
    import numpy as np, torch
    from paper_2103_03074_b200 import _lib
    lib = _lib.load()
    shape = [int(x) for x in os.environ.get("EXP_SHAPE", "15,12,15").split(",")]
    M, N, K = (1 << shape[0]), (1 << shape[1]), (1 << shape[2])
    A = torch.randn(M, K, dtype=torch.complex64, device="cuda")
    B = torch.randn(K, N, dtype=torch.complex64, device="cuda")
    C = torch.empty(M, N, dtype=torch.complex64, device="cuda")
    # time the GEMM kernel alone: a head program would stage once; here the
    # tnb_cgemm call stages + multiplies, so time K=0-work baseline separately
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ts = []
    for it in range(7):
        ev[0].record()
        _lib.check(lib.tnb_cgemm(0, M, N, K, A.data_ptr(), B.data_ptr(), C.data_ptr(), 1, 1))
        ev[1].record(); ev[1].synchronize()
        if it >= 2: ts.append(ev[0].elapsed_time(ev[1]))
    ts.sort()
    print(json.dumps({"skip": os.environ.get("TNB_EXP_SKIP", "0"), "ms_min": ts[0], "ms_med": ts[len(ts)//2]}))
else:
    for sk in ["0", "3", "0", "3", "1", "2"]:
        env = dict(os.environ, TNB_EXP_SKIP=sk)
        smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader", "-lms", "200"],
                               stdout=subprocess.PIPE, text=True)
        out = subprocess.run([sys.executable, __file__, "run"], env=env, capture_output=True, text=True)
        smi.terminate()
        samples = smi.communicate()[0].strip().splitlines()
        print(out.stdout.strip(), out.stderr.strip()[-300:], "clocks/power samples (last 8):", samples[-8:])
