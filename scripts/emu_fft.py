import numpy as np
W = np.exp(2j*np.pi*np.arange(512)/512)
def rev3(k): return ((k&1)<<2)|(k&2)|((k>>2)&1)
def dft8(x):
    x = list(x); r = 0.70710678118654752440
    for m in range(4):
        a,b = x[m], x[m+4]; x[m] = a+b; d = a-b
        x[m+4] = [d, d*(1+1j)*r, d*1j, d*(-1+1j)*r][m]
    for h in (0,4):
        for m in range(2):
            a,b = x[h+m], x[h+m+2]; x[h+m] = a+b; d=a-b
            x[h+m+2] = d if m==0 else d*1j
    for h in range(0,8,2):
        a,b = x[h],x[h+1]; x[h]=a+b; x[h+1]=a-b
    return x
def fft512(z):
    # thread t holds x[m] = z[t+64m]
    X = [[z[t+64*m] for m in range(8)] for t in range(64)]
    S0 = {}; S1 = {}
    for t in range(64):
        x = dft8(X[t]); j0, j1 = t&7, t>>3
        for k2 in range(8):
            y = x[rev3(k2)]
            if k2: y = y*W[(t*k2)&511]
            S0[j0*65+k2*8+j1] = y
    for t in range(64):
        j0,k2 = t&7, t>>3
        x = dft8([S0[j0*65+k2*8+j1] for j1 in range(8)])
        for k1 in range(8):
            y = x[rev3(k1)]
            if k1: y = y*W[(8*j0*k1)&511]
            S1[k2*65+k1*8+j0] = y
    out = np.zeros(512, complex)
    for t in range(64):
        k2,k1 = t&7, t>>3
        y = dft8([S1[k2*65+k1*8+j0] for j0 in range(8)])
        for k0 in range(8): out[t+64*k0] = y[rev3(k0)]
    return out
