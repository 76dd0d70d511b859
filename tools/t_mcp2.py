import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2010_12056_b200 as cpd
cpd.load_library()
rng = np.random.default_rng(0)
pre, K, post, R = [int(x) for x in sys.argv[1].split(',')] if len(sys.argv) > 1 else (3, 64, 200, 8)
Tn = rng.standard_normal((pre, K, post)); A = rng.standard_normal((K, R))
T = torch.from_numpy(Tn).cuda(); Ad = torch.from_numpy(A).cuda()
ref = np.einsum('pkm,kr->pmr', Tn, A).reshape(pre * post, R)
for trial in range(3):
    out = torch.full((pre * post, R), float('nan'), dtype=torch.float64, device='cuda')
    cpd.cpd_ttm_i8(T, pre, K, post, Ad, R, out, use_digits=True)
    o = out.cpu().numpy()
    bad = np.where(np.abs(o - ref).max(axis=1) > 1e-8 * np.abs(ref).max())[0]
    print('trial', trial, 'bad', bad)
    for b in bad[:3]:
        # which ref row (if any) do we match?
        d = np.abs(ref - o[b]).max(axis=1)
        j = int(np.argmin(d))
        # partial sums: does o[b] equal the product over only some k?
        print(' row', b, 'closest ref row', j, 'dist %.2e' % d[j], 'o/ref ratio', (o[b] / ref[b])[:3])
