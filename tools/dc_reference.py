"""NumPy transcription of the divide-and-conquer steps of csrc/heevd.inc + tridiag.cuh (tearing,
xLAED2 deflation, bisection relative to the nearer pole, Gu-Eisenstat z, eigenvector columns), used
to check the algorithm on random tridiagonals before the GPU port.  Design aid, not the oracle:
python tools/dc_reference.py"""
import numpy as np
eps=1.1102230246251565e-16
def dc(d,e):
    n=len(d)
    Z=np.eye(n)
    dh=np.array([d[i]-(e[i-1] if i>0 else 0)-(e[i] if i<n-1 else 0) for i in range(n)])
    blocks=[(i,1) for i in range(n)]
    while len(blocks)>1:
        nxt=[]; Z2=Z.copy(); newd=dh.copy()
        for b in range(0,len(blocks),2):
            if b+1>=len(blocks):
                nxt.append(blocks[b]); continue
            s,k1=blocks[b]; k=k1+blocks[b+1][1]; nxt.append((s,k))
            z=np.array([Z[s+k1-1,s+i] if i<k1 else Z[s+k1,s+i] for i in range(k)])
            beta=e[s+k1-1]; rho=2*beta
            dl=dh[s:s+k].copy(); zl=z*0.7071067811865476
            flip=rho<0
            if flip: rho=-rho; dl=-dl
            ord_=sorted(range(k),key=lambda i:dl[i])
            tol=8*eps*max(np.max(np.abs(dl)),rho*np.max(np.abs(zl)))
            keep=[];defl=[];pj=-1; rots=[]
            for nj in ord_:
                if rho*abs(zl[nj])<=tol: defl.append(nj); continue
                if pj<0: pj=nj; continue
                sg=zl[pj]; c=zl[nj]; tau=np.hypot(c,sg); t=dl[nj]-dl[pj]; c/=tau; sg=-sg/tau
                if abs(t*c*sg)<=tol:
                    zl[nj]=tau; zl[pj]=0; rots.append((pj,nj,c,sg))
                    tt=dl[pj]*c*c+dl[nj]*sg*sg; dl[nj]=dl[pj]*sg*sg+dl[nj]*c*c; dl[pj]=tt
                    defl.append(pj); pj=nj
                else:
                    keep.append(pj); pj=nj
            if pj>=0: keep.append(pj)
            keep=sorted(keep,key=lambda i:dl[i])
            Zb=Z[s:s+k,s:s+k].copy()
            for (a,bb,c,sg) in rots:
                x=Zb[:,a].copy(); y=Zb[:,bb].copy(); Zb[:,a]=c*x+sg*y; Zb[:,bb]=c*y-sg*x
            kk=len(keep); D=np.array([dl[i] for i in keep]); zz=np.array([zl[i] for i in keep])
            ZZ=np.sum(zz*zz)
            org=np.zeros(kk,int); taus=np.zeros(kk); lam=np.zeros(kk)
            for m in range(kk):
                lo=D[m]; hi=D[m+1] if m+1<kk else D[-1]+rho*ZZ
                f=lambda o,t: 1+rho*np.sum(zz*zz/((D-D[o])-t))
                mid=0.5*(hi-lo); o=m
                if m+1<kk and f(m,mid)<0: o=m+1; a=-mid; b_=0.0
                else: a=0.0; b_=mid if m+1<kk else hi-lo
                for it in range(200):
                    t=0.5*(a+b_)
                    if t==a or t==b_: break
                    fv=f(o,t)
                    if fv<0: a=t
                    elif fv>0: b_=t
                    else: a=b_=t; break
                t=0.5*(a+b_); org[m]=o; taus[m]=t; lam[m]=D[o]+t
            zh=np.zeros(kk)
            for i in range(kk):
                p=((D[org[kk-1]]-D[i])+taus[kk-1])/rho
                for m in range(kk-1):
                    num=(D[org[m]]-D[i])+taus[m]; den=(D[m]-D[i]) if m<i else (D[m+1]-D[i])
                    p*=num/den
                zh[i]=np.copysign(np.sqrt(abs(p)),zz[i])
            U=np.zeros((kk,kk))
            for m in range(kk):
                u=zh/((D-D[org[m]])-taus[m]); U[:,m]=u/np.linalg.norm(u)
            newZ=np.zeros((k,k))
            newZ[:,:kk]=Zb[:,keep]@U
            for t,cidx in enumerate(defl): newZ[:,kk+t]=Zb[:,cidx]
            Z2[s:s+k,s:s+k]=newZ
            nd=np.concatenate([lam, [dl[c] for c in defl]])
            if flip: nd=-nd
            newd[s:s+k]=nd
        Z=Z2; dh=newd; blocks=nxt
    return dh,Z
rng=np.random.default_rng(0)
for n in [2,3,7,16,33,64,100]:
    d=rng.standard_normal(n); e=rng.standard_normal(n-1)
    T=np.diag(d)+np.diag(e,1)+np.diag(e,-1)
    w,Z=dc(d,e)
    ref=np.linalg.eigvalsh(T)
    print(n, np.max(np.abs(np.sort(w)-ref)), np.linalg.norm(T@Z-Z*w), np.linalg.norm(Z.T@Z-np.eye(n)))
