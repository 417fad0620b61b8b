import itertools
def wavefronts(addrs, f):
    # addrs: list of 32 element indices (complex, 16 B) for a warp; returns wavefronts for LDS.128
    w = 0
    for ph in range(4):
        slots = {}
        for a in addrs[ph*8:(ph+1)*8]:
            if a is None: continue
            fa = f(a)
            slots.setdefault(fa % 8, set()).add(fa)
        w += max((len(s) for s in slots.values()), default=0)
    return w
def stage_patterns(L1, T=256):
    l = L1.bit_length()-1; S4 = l//2; pats = []
    for s in range(S4):
        lm = 2*(s+1); lmp = lm-2; mprev = 1<<lmp
        nb = L1//4
        for j in range(4):
            for w0 in range(0, min(nb,T), 32):
                addrs=[]
                for b in range(w0, w0+32):
                    if b >= nb: addrs.append(None); continue
                    k = b & (mprev-1); base = ((b>>lmp)<<lm)+k
                    addrs.append(base + j*mprev)
                pats.append(('r4', lm, addrs))
    if l & 1:
        mprev = L1//2; nb=L1//2
        for j in range(2):
            for w0 in range(0, min(nb,T), 32):
                addrs=[]
                for b in range(w0,w0+32):
                    k = b & (mprev-1); base = ((b>>(l-1))<<l)+k
                    addrs.append(base+j*mprev)
                pats.append(('r2', l, addrs))
    # consecutive element loops
    for w0 in range(0, min(L1,T), 32):
        pats.append(('lin',0,list(range(w0,w0+32))))
    return pats
cands = {
 'none': lambda p: p,
 'p+p>>4': lambda p: p + (p>>4),
 'p+p>>3': lambda p: p + (p>>3),
 'xor3': lambda p: p ^ ((p>>3)&7),
 'xor2': lambda p: p ^ ((p>>2)&7),
 'xor_mix': lambda p: p ^ (((p>>3) ^ (p>>5)) & 7),
 'xor_mix2': lambda p: p ^ (((p>>2) ^ (p>>4)) & 7),
 'xor_mix3': lambda p: p ^ (((p>>2) ^ (p>>4)^(p>>6)) & 7),
 'p+p>>2+p>>4': lambda p: p + (p>>2),
}
for L1 in (256, 512, 1024, 2048, 4096):
    pats = stage_patterns(L1)
    print(L1, end=': ')
    for nm, f in cands.items():
        tot = sum(wavefronts(a, f) for _,_,a in pats); ideal = sum(wavefronts(a, lambda p: p) if False else 4 for _,_,a in pats)
        print(f"{nm}={tot/ideal:.2f}", end='  ')
    print()

def perm_of(L1):
    l = L1.bit_length()-1
    radices = [4]*(l//2) + ([2] if l & 1 else [])
    perm = []
    for i in range(L1):
        x = i; digits = []
        for r in radices: digits.append(x % r); x //= r
        # perm[i] = sum d_s prod_{t>s} r_t
        v = 0
        for s, d in enumerate(digits):
            prod = 1
            for t in range(s+1, len(radices)): prod *= radices[t]
            v += d*prod
        perm.append(v)
    return perm
def col_k1(L1, C, r, col):
    pi = r + (col >> 1)*C
    if pi == 0: return L1//2 if (col & 1) else 0
    return L1 - pi if (col & 1) else pi
def slot_table(L1):
    perm = perm_of(L1)   # slot p holds X[perm[p]] -> slot of bin k = inverse perm
    inv = [0]*L1
    for p,k in enumerate(perm): inv[k] = p
    return inv
def cross_patterns(L1, C, T=256):
    slot = slot_table(L1); ncol = L1//C; pats=[]
    for r in range(C):
        for w0 in range(0, min(L1,T), 32):
            addrs=[]
            for u in range(w0, w0+32):
                q, col = divmod(u, ncol)
                addrs.append(slot[col_k1(L1, C, q, col)])
            pats.append(addrs)
    return pats
def pass16_patterns(L1, T=256):
    l = L1.bit_length()-1; S4 = l//2; npair = S4//2; pats=[]
    for i in range(npair):
        lm = 4*i+4; lmpp = lm-4; mp = 1<<(lm-2); mpp = 1<<lmpp
        nsb = L1>>4
        for j in range(4):
            for jp in range(4):
                for w0 in range(0, min(nsb,T), 32):
                    addrs=[]
                    for u in range(w0,w0+32):
                        if u >= nsb: addrs.append(None); continue
                        kpp = u & (mpp-1); base = ((u>>lmpp)<<lm)+kpp
                        addrs.append(base + j*mp + jp*mpp)
                    pats.append(addrs)
    return pats
for L1, C in ((1024,16),(512,16),(512,2),(256,2),(4096,1),(2048,8),(8192,16)):
    print(L1, C, end=': ')
    for nm in ('none','p+p>>4','xor2','xor_mix2'):
        f = cands[nm]
        cp = cross_patterns(L1, C); pp = pass16_patterns(L1)
        c = sum(wavefronts(a,f) for a in cp)/(4*len(cp))
        p = sum(wavefronts(a,f) for a in pp)/(4*max(len(pp),1))
        print(f"{nm}: cross={c:.2f} p16={p:.2f}", end='  ')
    print()

def brev32(x): return int('{:032b}'.format(x)[::-1], 2)
def rev4(x, m):
    if m == 0: return 0
    y = brev32(x) >> (32 - 2*m)
    return ((y & 0x55555555) << 1) | ((y >> 1) & 0x55555555)
def dperm(p, l):
    S4 = l//2
    if l % 2 == 0: return rev4(p, S4)
    return 2*rev4(p & ((1 << 2*S4)-1), S4) + (p >> (2*S4))
def dslot(k, l):
    S4 = l//2
    if l % 2 == 0: return rev4(k, S4)
    return rev4(k >> 1, S4) + ((k & 1) << (2*S4))
for l in range(1, 14):
    L = 1 << l; pm = perm_of(L); sl = slot_table(L)
    assert all(dperm(p, l) == pm[p] for p in range(L)), l
    assert all(dslot(k, l) == sl[k] for k in range(L)), l
print("perm formulas ok")
