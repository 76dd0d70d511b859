"""Ad-hoc check of the int8 TTM layouts against NumPy (digits vs converting path)."""
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2010_12056_b200 as cpd
cpd.load_library()
rng = np.random.default_rng(0)
cases = [tuple(int(x) for x in c.split(',')) for c in sys.argv[1:]] or [(40, 64, 256, 8), (40, 64, 384, 8), (40, 64, 192, 8), (1, 64, 192, 8), (3, 64, 72, 8), (1, 64, 72, 8), (2, 64, 144, 8), (40, 200, 200, 8)]
for (pre, K, post, R) in cases:
    Tn = rng.standard_normal((pre, K, post))
    A = rng.standard_normal((K, R))
    T = torch.from_numpy(Tn).cuda(); Ad = torch.from_numpy(A).cuda()
    out = torch.full((pre * post, R), float('nan'), dtype=torch.float64, device='cuda')
    ref = np.einsum('pkm,kr->pmr', Tn, A).reshape(pre * post, R)
    cpd.cpd_ttm_i8(T, pre, K, post, Ad, R, out, use_digits=True)
    o = out.cpu().numpy()
    err = np.linalg.norm(o - ref) / np.linalg.norm(ref)
    bad = np.where(np.abs(o - ref).max(axis=1) > 1e-8 * np.abs(ref).max())[0]
    nan = np.isnan(o).any(axis=1)
    print(pre, K, post, R, '%.2e' % err, 'bad rows', len(bad), bad[:6], 'unwritten', int(nan.sum()), np.where(nan)[0][:6], 'zero rows', int((np.abs(o).max(axis=1) == 0).sum()), flush=True)
