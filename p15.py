import numpy as np
from hear.ckks.encoder import Embedding, encode_coeffs
# compare reference fp64 encode against extended-precision (longdouble) FFT of same math
for n, logscale in [(1<<14,31),(1<<14,35),(1<<15,31),(1<<16,40),(1<<16,50)]:
    emb=Embedding(n); rng=np.random.default_rng(3)
    tot=0; mism=0; maxd=0
    for trial in range(4):
        v=rng.uniform(-1,1,n//2)
        ref=encode_coeffs(emb,v,float(1<<logscale))
        spec=np.zeros(2*n,dtype=np.clongdouble)
        spec[emb.rot_group]=v; spec[emb.conj_group]=v
        hp=np.fft.fft(spec)[:n].real/n*np.longdouble(1<<logscale)
        hpi=np.rint(hp).astype(np.int64)
        d=np.abs(hpi-ref); mism+=(d>0).sum(); maxd=max(maxd,d.max()); tot+=n
    print(f"N=2^{n.bit_length()-1} scale=2^{logscale}: coeff mismatches vs longdouble {mism}/{tot}  max|diff|={maxd}  max|coeff|~2^{np.log2(np.abs(ref).max()):.1f}")
print("longdouble eps", np.finfo(np.longdouble).eps)
