# Shared-memory wavefront model of plane_kernel_g (csrc/ldg_fused.cu) for hex
# p = 1, 2: per-thread 8-B and broadcast 16-B accesses of the main stages,
# wavefronts = max distinct 4-B words per bank; searches the plane / row /
# slot strides and the element stride.  python scripts/plane_banks.py N1
import itertools, sys
def wf(addrs_words):
    # addrs_words: list of sets of 4B word addresses per lane
    banks = {}
    for ws in addrs_words:
        for w in ws:
            banks.setdefault(w % 32, set()).add(w)
    return max(len(v) for v in banks.values()) if banks else 0
def acc8(dbl_addrs):   # per-lane double addresses (None = inactive)
    return wf([{2*a, 2*a+1} for a in dbl_addrs if a is not None])
def acc16(dbl_addrs):
    return wf([{2*a, 2*a+1, 2*a+2, 2*a+3} for a in dbl_addrs if a is not None])
def cost(N1, PS, PER, skew, ES, XS, inbuf):
    NP=N1*N1; EPW=32//N1
    lanes=[(l//N1, l%N1) for l in range(32)]
    def base(ls): return ls*PER + (ls>>2)*skew
    tot=0
    for cur in range(2):
        b0=cur*inbuf
        # up loads per-thread
        for n in range(NP): tot+=acc8([base(ls)+b0+k*PS+n for ls,k in lanes])
        # broadcast plane reads (planes m), pairs
        for m in range(N1):
            off=m*PS; H=(b0+off)&1
            tot+=acc8([base(ls)+b0+off for ls,k in lanes]) if H else 0
            for j in range((NP-H)//2): tot+=acc16([base(ls)+b0+off+H+2*j for ls,k in lanes])
            if (NP-H)&1: tot+=acc8([base(ls)+b0+off+NP-1 for ls,k in lanes])
        # W / out per-thread writes twice, planes read again (stage F) -> weight
        for n in range(NP): tot+=2*acc8([base(ls)+b0+k*PS+n for ls,k in lanes])
        for m in range(N1):
            off=m*PS; H=(b0+off)&1
            tot+=acc8([base(ls)+b0+off for ls,k in lanes]) if H else 0
            for j in range((NP-H)//2): tot+=acc16([base(ls)+b0+off+H+2*j for ls,k in lanes])
            if (NP-H)&1: tot+=acc8([base(ls)+b0+off+NP-1 for ls,k in lanes])
    tot/=2
    OffJ=2*inbuf; OffE=OffJ+4*N1*ES
    # jumps per thread writes (2 arrays)
    for f in range(2):
        for i in range(N1): tot+=2*acc8([base(ls)+OffJ+f*N1*ES+k*ES+i for ls,k in lanes])
    # T2 per-thread writes + reads of broadcast sJZ
    for n in range(NP):
        tot+=acc8([base(ls)+OffE+k*PS+n for ls,k in lanes])
        tot+=2*acc8([base(ls)+OffJ+(n//N1)*ES+n%N1 for ls,k in lanes])
        tot+=2*acc8([base(ls)+OffJ+2*N1*ES+(n//N1)*ES+n%N1 for ls,k in lanes])  # sFZ stage E
    # T2 planes broadcast read (stage E)
    for m in range(N1):
        off=OffE+m*PS; H=off&1
        tot+=acc8([base(ls)+off for ls,k in lanes]) if H else 0
        for j in range((NP-H)//2): tot+=acc16([base(ls)+off+H+2*j for ls,k in lanes])
        if (NP-H)&1: tot+=acc8([base(ls)+off+NP-1 for ls,k in lanes])
    # z-face column reads fzp + sFZ RMW
    for f in range(2):
        for j in range(N1):
            tot+=acc8([base(ls)+OffE+(f*(N1-1))*PS+k+N1*j for ls,k in lanes])
            tot+=2*acc8([base(ls)+OffJ+2*N1*ES+f*N1*ES+j*ES+k for ls,k in lanes])
    OffXY=OffE+N1*PS
    for idx in range(4*N1): tot+=5*acc8([base(ls)+OffXY+k*XS+idx for ls,k in lanes])
    return tot
if __name__=="__main__":
    N1=int(sys.argv[1]); NP=N1*N1
    res=[]
    for PS in range(NP+1, NP+8):
        for ES in range(N1, N1+4):
            for XS in range(4*N1, 4*N1+6):
                inb0=N1*PS+((N1*PS)&1)+28
                for inbuf in (inb0, inb0+2, inb0+4, inb0+6):
                    raw=2*inbuf+4*N1*ES+N1*PS+N1*XS
                    for pad in range(0,16,2):
                        PER=raw+pad+(raw&1)
                        for skew in (0,2,4,6,8,10):
                            res.append((cost(N1,PS,PER,skew,ES,XS,inbuf), PER, PS, ES, XS, inbuf, skew))
    res.sort()
    cur=[r for r in res if r[2]==NP+1 and r[3]==N1+1 and r[4]==4*N1+1 and r[6]==2]
    print("best", res[:8]); print("current-like", [c for c in cur if c[1]%16==4][:3])
