"""What-if: does tensor-core power (hence the power-capped clock) depend on
the bit activity of the fp16 lo planes?  Times the top C4 GEMM shape via
tnb_cgemm with lo zeroed / mantissa-truncated (TNB_EXP_LO_MASK; diagnostic)."""
import os, sys, subprocess, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1:
    import torch
    from paper_2103_03074_b200 import _lib
    lib = _lib.load()
    M, N, K = 1 << 15, 1 << 12, 1 << 15
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn(M, K, dtype=torch.complex64, device="cuda", generator=g)
    B = torch.randn(K, N, dtype=torch.complex64, device="cuda", generator=g)
    C = torch.empty(M, N, dtype=torch.complex64, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ts = []
    for it in range(6):
        ev[0].record()
        _lib.check(lib.tnb_cgemm(0, M, N, K, A.data_ptr(), B.data_ptr(), C.data_ptr(), 1, 1))
        ev[1].record(); ev[1].synchronize()
        if it >= 2: ts.append(ev[0].elapsed_time(ev[1]))
    ref = (A[:256].to(torch.complex128) @ B.to(torch.complex128))
    err = float(torch.linalg.norm(C[:256].to(torch.complex128) - ref) / torch.linalg.norm(ref))
    print(json.dumps({"mask": os.environ.get("TNB_EXP_LO_MASK", "none"), "ms_min": min(ts), "ms_med": sorted(ts)[len(ts)//2], "rel_err": err}))
else:
    # fp16: sign 1 | exp 5 | mantissa 10 ; masks keep the top k mantissa bits of both halves
    for m in [None, "0x0", "0xFFE0FFE0", "0xFFF8FFF8", None]:
        env = dict(os.environ)
        if m: env["TNB_EXP_LO_MASK"] = m
        smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader", "-lms", "100"], stdout=subprocess.PIPE, text=True)
        out = subprocess.run([sys.executable, __file__, "run"], env=env, capture_output=True, text=True)
        smi.terminate()
        samples = smi.communicate()[0].strip().splitlines()
        busy = [s for s in samples if float(s.split(",")[1].split()[0]) > 700]
        print(out.stdout.strip(), out.stderr.strip()[-300:], "| busy samples:", busy[-4:])
