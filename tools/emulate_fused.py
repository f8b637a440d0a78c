# Design probe (not product, not oracle): fp32 numpy emulation of the fused
# stale-shift kernel arithmetic and summation tree, compared with the golden
# reference fixtures. Usage: python tools/emulate_fused.py g1_c1_n1024
# faithful fp32 emulation of the planned fused kernel's arithmetic + summation structure
import sys, numpy as np, time
sys.path.insert(0,'oracle'); import lsk_oracle as O
f32=np.float32; f64=np.float64
L2E=f32(1.4426950408889634)
def ex2(t): return np.exp2(t.astype(f64)).astype(f32)
def eshift(x, sl2e): return ex2((x.astype(f64)*f64(L2E)-sl2e.astype(f64)).astype(f32))
def butterfly(v):  # v (..., 32) -> (...,) identical-lane xor butterfly sum
    v=v.copy()
    for o in [16,8,4,2,1]:
        idx=np.arange(32)^o; v=(v+v[...,idx]).astype(f32)
    return v[...,0]
def block_sum(E, NT):  # E (R, W) per-element terms, columns j = 4(v*NT+t)+q
    R,W=E.shape; V=W//(4*NT)
    T=E.reshape(R,V,NT,4).transpose(0,2,1,3).reshape(R,NT,V*4)  # per thread (v,q) order
    acc=np.zeros((R,NT),f32)
    for k in range(V*4): acc=(acc+T[:,:,k]).astype(f32)
    NW=NT//32; w=butterfly(acc.reshape(R,NW,32))
    pad=np.zeros((R,32),f32); pad[:,:NW]=w
    return butterfly(pad)
def emu(C64, mu_w, nu_w, eps, K, G=148):
    C=C64.astype(f32); n,m=C.shape
    NT,V = (256,1) if m<=1024 else (512,1) if m<=2048 else (512,2) if m<=4096 else (512,4)
    W=4*V*NT
    Cp=np.zeros((n,W),f32); Cp[:,:m]=C
    lmu=np.log(mu_w).astype(f32); lnu=np.full(W,-np.inf,f32); lnu[:m]=np.log(nu_w).astype(f32)
    inv=f32(1)/f32(eps); neg=-f32(eps)
    f=np.zeros(n,f32); g=np.zeros(W,f32)
    bounds=[(b*n//G,(b+1)*n//G) for b in range(G)]
    fires=[0,0]
    for k in range(1,K+1):
        X=(((g[None,:]-Cp)*inv).astype(f32)+lnu[None,:]).astype(f32)
        if k==1: M=X.max(1)
        else: M=(-f*inv).astype(f32)
        S=block_sum(eshift(X,(M*L2E).astype(f32)[:,None]),NT)
        bad=~((S>=1e-20)&(S<=1e30))
        if bad.any():
            fires[0]+=int(bad.sum()); M2=X.max(1); S2=block_sum(eshift(X,(M2*L2E).astype(f32)[:,None]),NT)
            M=np.where(bad,M2,M); S=np.where(bad,S2,S)
        f=(neg*(M+np.log(np.maximum(S,f32(1e-30))).astype(f32))).astype(f32)
        Y=(((f[:,None]-Cp)*inv).astype(f32)+lmu[:,None]).astype(f32)
        s=(-g*inv).astype(f32)
        Ey=eshift(Y,(s*L2E).astype(f32)[None,:])
        fwd=(k%2==1)
        P=np.zeros((G,W),f32)
        maxlen=max(r1-r0 for r0,r1 in bounds)
        for t in range(maxlen):
            for b,(r0,r1) in enumerate(bounds):
                if t<r1-r0:
                    i=r0+t if fwd else r1-1-t
                    P[b]=(P[b]+Ey[i]).astype(f32)
        # combine: 16 warps each sum a contiguous range of b sequentially, then butterfly over 32 slots
        NWc=16; parts=np.zeros((32,W),f32)
        for w in range(NWc):
            b0,b1=w*G//NWc,(w+1)*G//NWc
            acc=np.zeros(W,f32)
            for b in range(b0,b1): acc=(acc+P[b]).astype(f32)
            parts[w]=acc
        T=butterfly(parts.T)
        bad=~((T>=1e-20)&(T<=1e30))
        if bad.any():
            fires[1]+=1
            M2=Y.max(0); T2=Ey2=eshift(Y,(M2*L2E).astype(f32)[None,:]).sum(0,dtype=f64).astype(f32)  # exact path (approx structure)
            s=np.where(bad,M2,s); T=np.where(bad,T2,T)
        g=(neg*(s+np.log(np.maximum(T,f32(1e-30))).astype(f32))).astype(f32)
        g[m:]=0
    return f,g[:m],fires
for name in sys.argv[1:]:
    z=np.load(f'tests/golden/{name}.npz')
    n=int(z['n']); d=int(z['d']); X,Y=O.uniform_points(n,d,0); C64=O.sq_euclidean_cost(X,Y)
    t=time.time(); f,g,fires=emu(C64,z['mu'],z['nu'],float(z['eps']),int(z['K']))
    ra=np.abs(f-z['alpha']).max()/np.abs(z['alpha']).max(); rb=np.abs(g-z['beta']).max()/np.abs(z['beta']).max()
    print(name, fires, 'f rel',ra,'g rel',rb, 'gauge', (f-z['alpha']).mean(), time.time()-t)
