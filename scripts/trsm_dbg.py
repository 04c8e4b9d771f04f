import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2303_04353_b200 as casc
sys.path.insert(0, "tests")
m, n = 300, 70
rng = np.random.default_rng(13)
hi = np.tril(rng.uniform(-1, 1, (m, m)) / m); lo = hi * 2.0**-53 * rng.uniform(-1, 1, (m, m))
d = 1.0 + rng.uniform(0, 1, m); hi[np.arange(m), np.arange(m)] = d; lo[np.arange(m), np.arange(m)] = d * 2.0**-54
rng = np.random.default_rng(15)
B_hi = rng.uniform(-1, 1, (m, n)); B_lo = B_hi * 2.0**-53 * rng.uniform(-1, 1, (m, n))
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
def run(alpha, pad):
    wh = T(np.pad(B_hi, ((0, 0), (0, pad)))); wl = T(np.pad(B_lo, ((0, 0), (0, pad))))
    casc.casc_trsm_fp64x2("L", "N", alpha, T(hi), T(lo), wh[:, :n], wl[:, :n])
    return wh[:, :n].cpu().numpy(), wl[:, :n].cpu().numpy()
a = run(1.0, 0); b = run(1.0, 3); c = run(4.0, 0)
print("stride: hi eq", np.array_equal(a[0], b[0]), "lo eq", np.array_equal(a[1], b[1]), "ndiff", (a[1] != b[1]).sum())
print("alpha4: hi eq", np.array_equal(4 * a[0], c[0]), "lo eq", np.array_equal(4 * a[1], c[1]), "ndiff", (4 * a[1] != c[1]).sum())
idx = np.argwhere(4 * a[1] != c[1])[:5]
for i, j in idx: print(i, j, a[0][i, j], a[1][i, j] * 4, c[1][i, j])
# GEMM scaling check
A = T(hi[:64, :64]); Al = T(lo[:64, :64]); Bh = T(B_hi[:64]); Bl = T(B_lo[:64])
r1 = casc.casc_gemm_fp64x2(A, Al, Bh, Bl); r4 = casc.casc_gemm_fp64x2(A, Al, 4 * Bh, 4 * Bl)
print("gemm scale lo eq", torch.equal(4 * r1[1], r4[1]), "hi eq", torch.equal(4 * r1[0], r4[0]))
