"""Run tools/libtcprobe.so on random tf32-exact inputs and compare with an fp64 matmul."""
import ctypes, os, sys
import numpy as np, torch
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libtcprobe.so"))
lib.tc_probe.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int, ctypes.c_int]

def tf32(x):
    u = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x0FFF + ((u >> 13) & 1)) & 0xFFFFE000     # round to nearest even on 10 mantissa bits
    return u.astype(np.uint32).view(np.float32)

rng = np.random.default_rng(0)
for N in (128, 256):
    for K in (32, 96):
        A = tf32(rng.standard_normal((128, K)))
        B = tf32(rng.standard_normal((N, K)))
        dA, dB = torch.tensor(A).cuda(), torch.tensor(B).cuda()
        dD = torch.zeros((128, N), dtype=torch.float32, device="cuda")
        rc = lib.tc_probe(dA.data_ptr(), dB.data_ptr(), dD.data_ptr(), K, N)
        D = dD.cpu().numpy()
        ref = A.astype(np.float64) @ B.astype(np.float64).T
        err = np.abs(D - ref).max() / np.abs(ref).max()
        print(f"N={N} K={K} rc={rc} max rel err {err:.3e}", "OK" if err < 1e-5 else "FAIL")
        if err > 1e-5:
            bad = np.argwhere(np.abs(D - ref) > 1e-3 * np.abs(ref).max())
            print("  first bad", bad[:5], D[tuple(bad[0])], ref[tuple(bad[0])])
