p='/root/repo/paper_1901_01685_b200/csrc/cuda/skew.cu'
s=open(p).read()
s=s.replace("""__device__ __forceinline__ void st_shared_if(double* p, double v, bool pred) {""","""__device__ __forceinline__ double ld_shared_f64(const char* p) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(smem_u32(p)));
    return v;
}
__device__ __forceinline__ void st_shared_if(double* p, double v, bool pred) {""")
old="""        auto group_wait = [&](unsigned q) {  // items and right-hand sides of group q are in"""
new="""        auto fetch_w = [&](int t, Pre& f) {  // coefficients / rhs of step t
            const uint4* it = &sm.item[t & (PF - 1)][0][lane];
            const uint4 c0 = it[0], c1 = it[32];
            f.w[0] = __hiloint2double(int(c0.y), int(c0.x));
            f.w[1] = __hiloint2double(int(c0.w), int(c0.z));
            f.w[2] = __hiloint2double(int(c1.y), int(c1.x));
            f.w[3] = __hiloint2double(int(c1.w), int(c1.z));
            f.rhs = sm.rhs[t & (PF - 1)][lane];
            if (K == kSkewGS) f.su = sm.su[t & (PF - 1)][lane];
        };
        auto fetch_o = [&](int t, int (&o)[4]) {  // value offsets of step t
            const uint4 c2 = sm.item[t & (PF - 1)][2][lane];
            o[0] = int(c2.x);
            o[1] = int(c2.y);
            o[2] = int(c2.z);
            o[3] = int(c2.w);
        };
        auto group_wait = [&](unsigned q) {  // items and right-hand sides of group q are in"""
assert old in s; s=s.replace(old,new)
i=s.index("        double res = 0.0, xprev = 0.0;\n        int hr = INT_MIN / 2;  // last seen halo_ready")
j=s.index("        if (TR && a.trace && lane == 0) a.trace[blk * 8 + 1] = gtimer();\n")
new=open('/tmp/loop_body.txt').read()
s=s[:i]+new+s[j:]
old="""    int q = r.len - 1;
    if (q >= 0 && r.col(q) == v - 1 && ix > 0) --q;  // stage 0: the v-1 term
    int prev = INT_MAX;
    bool ok = true;"""
new="""    int q = r.len - 1;
    if (q >= 0 && r.col(q) == v - 1 && ix > 0) --q;  // stage 0: the v-1 and v-2 terms (registers)
    if (q >= 0 && r.col(q) == v - 2 && ix > 1) --q;
    int prev = INT_MAX;
    bool ok = true;"""
assert old in s; s=s.replace(old,new)
s=s.replace("""        if (d == 0 && st > ix - jx - 1) {  // own value not final by the stage's step""","""        if (d == 0 && st > ix - jx - 2) {  // own value not final a step before the stage's step""")
s=s.replace("""            const int need = st + 1 + jx - ix;  // d * D >= need for a term inside the block""","""            const int need = st + 2 + jx - ix;  // d * D >= need for a term inside the block""")
s=s.replace("""            Rl[hd] = max(Rl[hd], st + 1 + jx - ix - D * k);""","""            Rl[hd] = max(Rl[hd], st + 2 + jx - ix - D * k);""")
old="""        int q = r.len - 1;
        const bool has0 = q >= 0 && r.col(q) == v - 1 && ix > 0;
        if (role == 0) {
            it.w[0] = has0 ? r.val(q) : 0.0;
            it.w[1] = K == kSkewL ? 1.0 : dinv[v];
            it.o[0] = has0 ? 8 : 0;
        } else {
            if (has0) --q;"""
new="""        int q = r.len - 1;
        const bool has1 = q >= 0 && r.col(q) == v - 1 && ix > 0;
        const int q1 = has1 ? q - 1 : q;
        const bool has2 = q1 >= 0 && r.col(q1) == v - 2 && ix > 1;
        if (role == 0) {  // register terms: w[0] = a(v-1), w[2] = a(v-2), w[3] = flags
            it.w[0] = has1 ? r.val(q) : 0.0;
            it.w[1] = K == kSkewL ? 1.0 : dinv[v];
            it.w[2] = has2 ? r.val(q1) : 0.0;
            it.w[3] = double((has1 ? 1 : 0) | (has2 ? 2 : 0));
        } else {
            q = has2 ? q1 - 1 : q1;"""
assert old in s; s=s.replace(old,new)
s=s.replace("""//   stage 0     : w[0] = coefficient of the v-1 term, w[1] = 1/diagonal (U), o[0] = 8 if
//                 the row has a v-1 term else 0, o[1..3] = zero cell""","""//   stage 0     : w[0] / w[2] = coefficients of the v-1 / v-2 terms (taken from registers),
//                 w[1] = 1/diagonal (U, GS), w[3] = flags (1: v-1 present, 2: v-2 present),
//                 o[0..3] = zero cell""")
open(p,'w').write(s)
