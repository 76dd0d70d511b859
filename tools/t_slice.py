import sys, ctypes as C, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2010_12056_b200 as cpd
lib = cpd.load_library()
f = lib.cpd_debug_slice_digits
f.restype = C.c_int; f.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]
rng = np.random.default_rng(0)
for (rows, w) in [(192, 248), (192, 256), (128, 200), (3, 200)]:
    X = rng.standard_normal((rows, w))
    n = rows * w
    ipad = (w + 15) // 16 * 16
    ps = ((rows * ipad) + 63) // 64 * 64
    out = torch.full((7 * ps,), 77, dtype=torch.uint8, device='cuda')
    Xd = torch.from_numpy(X).cuda()
    assert f(Xd.data_ptr(), n, w, out.data_ptr(), None) == 0
    P = out.cpu().numpy().reshape(7, ps)[:, :rows * ipad].reshape(7, rows, ipad)
    # reconstruct values from digits
    dig = P.view(np.int8).astype(np.int64)
    v = sum(dig[a] * (256 ** a) for a in range(7))
    e = int(np.frexp(np.abs(X).max())[1])
    ref = np.rint(X * 2.0 ** (54 - e)).astype(np.int64)
    bad = np.argwhere(v[:, :w] != ref)
    padbad = np.argwhere(v[:, w:] != 0)
    print(rows, w, 'value mismatches', len(bad), bad[:5].tolist(), 'pad nonzero', len(padbad), padbad[:5].tolist(), flush=True)
