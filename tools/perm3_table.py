import itertools, numpy as np
f=np.float32
def zexpr(v):
    aa=f(v[0]+v[1]); bb=f(v[0]-v[1]); cc=f(v[2]+v[3]); dd=f(v[2]-v[3])
    return [f(aa-dd), f(bb+cc), f(bb-cc), f(-aa-dd)]
rng=np.random.default_rng(0)
V=[rng.standard_normal(4).astype(f) for _ in range(200)]
perms=list(itertools.permutations(range(4)))
# E: input perms Q with z_j(v∘Q) = eps_j z_{pi(j)}(v) bitwise
E={}
for Q in perms:
    ok=True; pi=None; eps=None
    for v in V:
        z=zexpr(v); zq=zexpr([v[Q[c]] for c in range(4)])
        p=[];e=[]
        for j in range(4):
            m=[(i,1) for i in range(4) if zq[j]==z[i] and np.signbit(zq[j])==np.signbit(z[i])]+[(i,-1) for i in range(4) if zq[j]==-z[i] and np.signbit(zq[j])!=np.signbit(z[i])]
            if len(m)!=1: ok=False;break
            p.append(m[0][0]); e.append(m[0][1])
        if not ok: break
        if pi is None: pi,eps=p,e
        elif pi!=p or eps!=e: ok=False;break
    if ok: E[Q]=(tuple(pi),tuple(eps))
print(len(E)); 
for Q,(pi,eps) in E.items(): print(Q,pi,eps)
Pi={pi for pi,_ in E.values()}
print("distinct pi",len(Pi))
# cosets: P[k] = pi(R[k])  => choose reps R_t
reps=[]
covered={}
for P in perms:
    if P in covered: continue
    reps.append(P)
    for Q,(pi,eps) in E.items():
        P2=tuple(pi[P[k]] for k in range(4))
        if P2 not in covered: covered[P2]=(len(reps)-1,Q,tuple(eps[P[k]] for k in range(4)))
print("reps",reps, len(covered))
# verify: X[k]=z_{P2[k]}(v) == sign * z_{R[k]}(v∘Q)
for P2,(t,Q,sg) in covered.items():
    R=reps[t]
    for v in V[:50]:
        z=zexpr(v); zq=zexpr([v[Q[c]] for c in range(4)])
        for k in range(4):
            a=z[P2[k]]; b=f(sg[k])*zq[R[k]]
            assert a==b and np.signbit(a)==np.signbit(b),(P2,t,Q,sg,k)
print("verified")
# emit table in the kernel's perm order: need PermAt<P,K> convention -> print by tuple
import json
json.dump({"reps":reps,"tab":{str(list(k)):[v[0],list(v[1]),list(v[2])] for k,v in covered.items()}},open("/tmp/sim/tab.json","w"))
