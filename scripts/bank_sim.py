# Offline shared-memory bank-conflict simulator for the Stockham exchange (see graf_fft.cuh).
def radices(M,E):
    RM=min(E,16); r=[]; m=M
    while m>=RM: r.append(RM); m//=RM
    return ([m] if m>1 else [])+r      # remainder first
def degree(addrs):
    worst=0
    for ph in range(0,len(addrs),16):
        b={}
        for a in set(addrs[ph:ph+16]): b.setdefault(a%16,set()).add(a)
        worst=max(worst,max(len(v) for v in b.values()))
    return worst
def sim(M,E,sh):
    pad=lambda y:y>>sh
    T=M//E; rad=radices(M,E); tot=0;cnt=0;worst=0; Ns=1
    stride=M+(M>>sh)
    for p,R in enumerate(rad[:-1]):
        Q=E//R
        for q in range(Q):
            for r in range(R):
                addrs=[]
                for lane in range(32):
                    sl=lane//T if T<32 else 0; t=lane%T if T<32 else lane
                    jp=t+q*T; y=(jp//Ns)*Ns*R+(jp%Ns)+r*Ns
                    addrs.append(sl*stride+pad(y)+y)
                d=degree(addrs); tot+=d;cnt+=1;worst=max(worst,d)
        for e in range(E):
            addrs=[]
            for lane in range(32):
                sl=lane//T if T<32 else 0; t=lane%T if T<32 else lane
                y=t+e*T; addrs.append(sl*stride+pad(y)+y)
            d=degree(addrs); tot+=d;cnt+=1;worst=max(worst,d)
        Ns*=R
    return (round(tot/cnt,3) if cnt else 0, worst)
for M,E in [(64,8),(128,16),(256,16),(512,8),(1024,16),(2048,16),(4096,16),(8192,16),(16384,16),(16384,32),(8192,32)]:
    print(M,E,radices(M,E),{s:sim(M,E,s) for s in (3,4,5)})
