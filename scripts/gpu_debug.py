import sys, numpy as np
sys.path.insert(0, '/root/repo')
sys.path.insert(0, '/tmp')
exec(open('/root/repo/scripts/emu_fft.py').read())
from oracle import oracle as O
from paper_1806_03461_b200 import tfhe
p = O.default_params(); K = O.Keys(p, 42); ctx = O.Context(p, K)
KK = tfhe.KeySet(seed=42); eng = tfhe.Engine(KK)
rng = np.random.default_rng(3)
polys = rng.integers(-64, 64, (4, 1024)).astype(np.int32).view(np.uint32)
got = eng.debug_fourier(polys)
psi = np.exp(1j*np.pi*np.arange(512)/1024)
for i in range(4):
    pl = polys[i].view(np.int32).astype(float)
    want = fft512((pl[:512] + 1j*pl[512:])*psi)/512
    print('fft poly', i, np.abs(got[i]-want).max())
bkf = eng.debug_fourier(count=12, which=1)
for r in range(6):
    for q in range(2):
        pl = K.bk[0, r, q].view(np.int32).astype(float)
        want = fft512((pl[:512] + 1j*pl[512:])*psi)/512
        print('bkf', r, q, np.abs(bkf[r*2+q]-want).max()/np.abs(want).max())
lwe = KK.encrypt(np.array([1], np.uint8), seed=11, stream=1)[0]
for it in (0, 1):
    g = eng.debug_blind_rotate(lwe, iters=it); w = ctx.blind_rotate(lwe, iters=it)
    d = (g.astype(np.int64) - w.astype(np.int64))
    print('iters', it, 'equal', np.array_equal(g, w), 'ndiff', np.count_nonzero(d), 'A', np.count_nonzero(d[:1024]), 'B', np.count_nonzero(d[1024:]))
    if it == 1 and not np.array_equal(g, w):
        print('first diffs idx', np.nonzero(d)[0][:20])
        print(g[:8], w[:8])
g = eng.debug_blind_rotate(lwe, iters=100001); w = ctx.blind_rotate(lwe, iters=1)
print('global-BK variant equal', np.array_equal(g, w))
