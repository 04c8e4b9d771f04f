"""Time experiment builds of the fused kernel (scripts/variants.py build|run)."""
import json, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
VARIANTS = {
    "base": [],
    "nocomb": ["CASC_EXPERIMENT_NO_COMBINE"],
    "bk16ns2": ["CASC_BK=16", "CASC_NSTAGE=2"],
    "bk8ns5": ["CASC_NSTAGE=5"],
    "bk4ns8": ["CASC_BK=4", "CASC_NSTAGE=8"],
    "pow2i": ["CASC_EXPERIMENT_POW2I"],
    "noinl": ["CASC_LDEXP_NOINLINE"],
    "always3": ["CASC_SCALE_ALWAYS3"],
}
if sys.argv[1] == "build":
    from paper_2303_04353_b200 import _build
    names = sys.argv[2:] or list(VARIANTS)
    for n in names:
        print(n, _build.build_variant(n, VARIANTS[n]), flush=True)
elif sys.argv[1] == "run":
    names = sys.argv[3:] or list(VARIANTS)
    n = int(sys.argv[2])
    for v in names:
        env = dict(os.environ, CASC_LIB_PATH=os.path.abspath(f"paper_2303_04353_b200/libcasc_{v}.so"))
        try:
            r = subprocess.run([sys.executable, __file__, "one", str(n)], env=env, capture_output=True, text=True, timeout=150)
        except subprocess.TimeoutExpired:
            print(v, "TIMEOUT", flush=True); continue
        print(v, r.stdout.strip(), r.stderr.strip()[-300:], flush=True)
elif sys.argv[1] == "one":
    import torch
    import paper_2303_04353_b200 as casc
    n = int(sys.argv[2])
    g = torch.Generator(device="cuda").manual_seed(0)
    A_hi = torch.rand(n, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    B_hi = torch.rand(n, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    A_lo = A_hi * 2.0**-54; B_lo = B_hi * 2.0**-54
    pa = casc.casc_pack_a(A_hi, A_lo); pb = casc.casc_pack_b(B_hi, B_lo)
    C = casc.casc_gemm_packed(n, n, n, pa, pb)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); casc.casc_gemm_packed(n, n, n, pa, pb, C_hi=C[0], C_lo=C[1], flags=C[2]); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    print(json.dumps({"n": n, "gemm_ms": ms, "tflops": 20 * n**3 / ms / 1e9, "frac": 20 * n**3 / ms / 1e9 / 37.109}))
