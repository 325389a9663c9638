// K1 fast path: k1_front + k1_mid fused for the common DAG, integer-only.
//
// For t_min = 1 and integer loads every quantity k1_front and k1_mid compute
// is an integer or an integer over M, so the whole front half of the
// analysis runs without a rational op (analysis.cpp:40-81 restated):
//   m^max(l) = l;  exec(l, min(l, M)) = 1 if l <= M else l/M  (units of 1/M:
//   w = max(M, l));  exec(l, m^max) = ceil(l/M);  graham_para = chain +
//   (U - chain)/M with U = sum l and chain = the longest path in nodes;
//   lower = max(U, weighted critical path in units of 1/M) / M.
// One warp per DAG (n <= 64: node v lives in lane v % 32, slot v / 32), and
// every phase is a uniform loop over k = 0..n-1 with the data of node k
// broadcast by a shuffle — no divergent per-lane loops:
//   closure     ids in topological order (every edge u < v): one pass in
//               index order folds anc[k] | {k} into k's successors (Warshall
//               in topological order), with the weighted prefix; the hop
//               level (longest path in nodes) by peeling sources layer by
//               layer, one ballot per layer (dag.cpp:69-124,
//               analysis.cpp:11-24);
//   W^anc       sum of the ancestors' loads (dag.cpp:126-135);
//   ranks       (W^anc desc, id asc) for heads/candidates, joins (W^anc asc,
//               id asc) (division.cpp:88-93, dag.cpp:218-230);
//   blocks      node v's block = the first join (in join order) it is an
//               ancestor of, else the residual (division.cpp:10-30);
//   division    a block's members form an in-block forest (one in-block
//               predecessor each); while no extraction truncates (<= M heads,
//               no oversized head next to others: Rules 1-2 of
//               division.cpp:94-113 idle), extraction i takes exactly the
//               members at in-block depth i, so division group = (block,
//               depth) in order, depth = |anc(v) ∩ block(v)|.
// Anything outside that case — fractional loads or t_min != 1 (batch-wide),
// n > 64, a load outside [1, 65535], an edge not in index order or out of
// range, not exactly one source and one sink, or a division layer that Rule 1
// or Rule 2 would cut — is queued (fb list) for the general kernels
// (k1_front / k1_mid), which reproduce every validation error and rule.
// The output is k1_mid's hand-off (K1Node, ro, divg, ndiv, shape key), so
// k1_back_lane walks both kinds of DAG alike.
#pragma once

namespace ds {

constexpr int kFastWarps = 4;
constexpr u64 kFastCounter = 6;    // retry_count[6]: next DAG of k1_fast<32>
constexpr u64 kFbCounter = 7;      // retry_count[7]: fallback list length
constexpr u64 kL64Counter = 8;     // retry_count[8]: DAGs with 32 < n <= 64 (list h.l64)
constexpr u64 kFast64Counter = 9;  // retry_count[9]: next entry of h.l64 for k1_fast<64>

struct FastWarp {
    u64 pred[64];          // edge scatter target
    unsigned int bdep[68]; // per block: max in-block depth + 1 (k1_fast<32>: layers)
    unsigned int gcnt[64]; // per division group: members
    unsigned int gbig[64]; // per division group: has an oversized member
    unsigned char ord[64]; // node at rank r
    unsigned char jord[32]; // k1_fast<32>: join at join position p
};

__device__ __forceinline__ u64 shfl64(u64 x, int src) {
    const u32 lo = __shfl_sync(FULL, u32(x), src), hi = __shfl_sync(FULL, u32(x >> 32), src);
    return (u64(hi) << 32) | lo;
}

// gcd of two positive u32 (binary)
__device__ __forceinline__ u32 fast_gcd(u32 a, u32 b) { return gcd32(a, b); }

// Returns DS_OK with the hand-off written, or -1: queue for the general path.
__device__ __forceinline__ int fast_dag(FastWarp& S, const K1Args& a, const int lane, const u64 d, const u32 n0,
                                        const int n, const u32 e0, const int ne, const int M) {
    if (n < 1 || n > 64) return -1;
    const bool hi = n > 32;
    const int va = lane, vb = lane + 32;
    const bool ina = va < n, inb = vb < n;
    u32 la, lb;
    u64 pa, pb;
    if (a.tri.adj) {  // triangular wire form: u16 loads, predecessor bits
        la = ina ? u32(a.tri.ln16[n0 + va]) : 1u;
        lb = inb ? u32(a.tri.ln16[n0 + vb]) : 1u;
        if (__any_sync(FULL, la < 1 || lb < 1)) return -1;
        const u32 w0 = a.tri.adj_off[d] - a.tri.adj_off[0], nw = a.tri.adj_off[d + 1] - a.tri.adj_off[d];
        pa = tri_preds(a.tri.adj + w0, nw, n, va);
        pb = hi ? tri_preds(a.tri.adj + w0, nw, n, vb) : 0ull;
    } else {
        // ---- loads: integers in [1, 65535]
        const long long la_ = ina ? (long long)a.load_num[n0 + va] : 1;
        const long long lb_ = inb ? (long long)a.load_num[n0 + vb] : 1;
        if (__any_sync(FULL, la_ < 1 || la_ > 65535 || lb_ < 1 || lb_ > 65535)) return -1;
        la = u32(la_);
        lb = u32(lb_);
        // ---- edges (sorted (from, to) words): all u < v < n, scattered to pred
        S.pred[lane] = 0;
        S.pred[lane + 32] = 0;
        __syncwarp();
        bool bad = false;
#pragma unroll 1
        for (int e = lane; e < ne; e += 32) {
            const u32 w = a.edges[e0 + e];
            const u32 u = w >> 16, v = w & 0xffffu;
            if (u >= v || v >= u32(n)) {
                bad = true;
            } else {
                atomicOr(reinterpret_cast<unsigned int*>(&S.pred[v]) + (u >> 5), 1u << (u & 31));
            }
        }
        if (__any_sync(FULL, bad)) return -1;
        __syncwarp();
        pa = S.pred[va];
        pb = hi ? S.pred[vb] : 0ull;
    }
    // ---- exactly one source and one sink (dag.cpp:97-108): in index order
    // node 0 is a source and node n-1 a sink, so check there are no others
    const u32 hs_lo = __reduce_or_sync(FULL, u32(pa) | u32(pb)), hs_hi = __reduce_or_sync(FULL, u32(pa >> 32) | u32(pb >> 32));
    const u64 has_succ = (u64(hs_hi) << 32) | hs_lo;
    const u64 V = n == 64 ? ~0ull : ((1ull << n) - 1);
    const u64 srcs = __ballot_sync(FULL, ina && pa == 0) | (u64(__ballot_sync(FULL, inb && pb == 0)) << 32);
    if (__popcll(srcs) != 1 || __popcll(V & ~has_succ) != 1) return -1;
    // ---- closure, hop level, weighted prefix (one pass in topological order)
    const bool flat = !__any_sync(FULL, (ina && la > u32(M)) || (inb && lb > u32(M)));
    const u32 wa = la > u32(M) ? la : u32(M), wb = lb > u32(M) ? lb : u32(M);  // exec in units of 1/M
    u64 aa = 0, ab = 0;     // ancestors
    u32 cpa = 0, cpb = 0;   // longest incoming weighted path (units of 1/M)
    // index order is topological, so node k < 32 has only ancestors < 32 (a
    // 32-bit word, one shuffle) and only slot-b nodes (v >= 32) can have a
    // predecessor k >= 32: two loops without per-k slot selects
    const int n1 = n < 32 ? n : 32;
    if (flat) {  // ancestors-or-self words, constant-k predecessor tests (cf. fast_dag32)
        u32 xa = ina ? (1u << va) : 0u;
        u64 xb = inb ? (1ull << vb) : 0ull;
#pragma unroll
        for (int k0 = 0; k0 < 32; k0 += 4) {
            if (k0 >= n1) break;
#pragma unroll
            for (int k = k0; k < k0 + 4; ++k) {
                const u32 ak = __shfl_sync(FULL, xa, k);
                if ((pa >> k) & 1) xa |= ak;
                if ((pb >> k) & 1) xb |= ak;
            }
        }
#pragma unroll
        for (int k0 = 32; k0 < 64; k0 += 4) {
            if (k0 >= n) break;
#pragma unroll
            for (int k = k0; k < k0 + 4; ++k) {
                const u64 ak = shfl64(xb, k - 32);
                if ((pb >> k) & 1) xb |= ak;
            }
        }
        aa = xa & ~(1u << va);
        ab = inb ? xb & ~(1ull << vb) : 0ull;
    } else {  // some load > M: the weighted prefix rides along
#pragma unroll 4
        for (int k = 0; k < n1; ++k) {
            const u32 ak = __shfl_sync(FULL, u32(aa), k) | (1u << k);
            const u32 ck = __shfl_sync(FULL, cpa + wa, k);
            if ((pa >> k) & 1) {
                aa |= ak;
                cpa = max(cpa, ck);
            }
            if ((pb >> k) & 1) {
                ab |= ak;
                cpb = max(cpb, ck);
            }
        }
#pragma unroll 4
        for (int k = 32; k < n; ++k) {
            const u64 ak = shfl64(ab, k - 32) | (1ull << k);
            const u32 ck = __shfl_sync(FULL, cpb + wb, k - 32);
            if ((pb >> k) & 1) {
                ab |= ak;
                cpb = max(cpb, ck);
            }
        }
    }
    // longest path in nodes: peel sources layer by layer (node v leaves in
    // round lv(v) + 1)
    u32 rounds64 = 0;
    for (u64 R = V; R; ++rounds64)
        R &= ~(u64(__ballot_sync(FULL, ina && ((R >> va) & 1) && !(pa & R))) |
               (u64(__ballot_sync(FULL, inb && ((R >> vb) & 1) && !(pb & R))) << 32));
    // ---- descendants: transpose of the ancestor matrix (dag.cpp:119-124)
    u64 da, db = 0;
    {
        const u32 t00 = warp_transpose32(u32(aa), lane);
        if (!hi) {
            da = t00;
        } else {
            const u32 t10 = warp_transpose32(u32(ab), lane), t01 = warp_transpose32(u32(aa >> 32), lane),
                      t11 = warp_transpose32(u32(ab >> 32), lane);
            da = (u64(t10) << 32) | t00;
            db = (u64(t11) << 32) | t01;
        }
    }
    // ---- bounds 1..4 (analysis.cpp:40-81)
    const u32 mask = a.mask;
    int64_t* bo = a.bounds + 10 * d;
    {
        const u32 U = __reduce_add_sync(FULL, (ina ? la : 0u) + (inb ? lb : 0u));
        const u32 GU = __reduce_add_sync(FULL, (ina ? (la + u32(M) - 1) / u32(M) : 0u) +
                                                   (inb ? (lb + u32(M) - 1) / u32(M) : 0u));
        const u32 G = flat ? u32(n) * u32(M) : __reduce_add_sync(FULL, (ina ? wa : 0u) + (inb ? wb : 0u));
        const u32 rounds = rounds64;  // longest path in nodes
        const u32 cp = flat ? rounds * u32(M)
                            : __reduce_max_sync(FULL, max(ina ? cpa + wa : 0u, inb ? cpb + wb : 0u));
        // lanes 0..3 reduce one bound each: greedy, greedy_unaware, graham_para, lower
        if (lane < 4) {
            const int k = lane + 1;
            u32 num = lane == 0 ? G : lane == 1 ? GU : lane == 2 ? rounds * u32(M) + U - rounds : (U > cp ? U : cp);
            u32 den = lane == 1 ? 1u : u32(M);
            const u32 g = fast_gcd(num, den);
            num /= g;
            den /= g;
            const bool want = mask & (1u << k);
            bo[2 * k] = want ? (long long)num : 0;
            bo[2 * k + 1] = want ? (long long)den : 0;
        }
    }
    const bool proposed = mask & DS_M_PROPOSED;
    if (!proposed) {
        if (lane < 2) bo[lane] = 0;
        if (lane == 0) {
            a.status[d] = DS_OK;
            if (a.n_groups) a.n_groups[d] = 0;
            if (a.h.skey) a.h.skey[d] = kWalkKeyNone;
        }
        return DS_OK;
    }
    // ---- W^anc = l + sum over ancestors, by load bit-planes (dag.cpp:126-135):
    // O(load bits) ballots instead of O(n) shuffles
    const int lbits = 32 - __clz(int(__reduce_or_sync(FULL, (ina ? la : 0u) | (inb ? lb : 0u))));
    u32 Wa = la, Wb = lb;
#pragma unroll 1
    for (int b = 0; b < lbits; ++b) {
        const u64 P = __ballot_sync(FULL, ina && ((la >> b) & 1)) |
                      (u64(__ballot_sync(FULL, inb && ((lb >> b) & 1))) << 32);
        Wa += u32(__popcll(aa & P)) << b;
        Wb += u32(__popcll(ab & P)) << b;
    }
    // ---- rank (W desc, id asc) and join position (W asc, id asc), bit-serial
    // over W's bits: eq* hold the nodes (joins) whose W agrees so far
    const u64 J = __ballot_sync(FULL, ina && __popcll(pa) >= 2) | (u64(__ballot_sync(FULL, inb && __popcll(pb) >= 2)) << 32);
    const int wbits = 32 - __clz(int(__reduce_or_sync(FULL, (ina ? Wa : 0u) | (inb ? Wb : 0u))));
    u64 eqra = V, eqrb = V, eqja = J, eqjb = J;
    int ra = 0, rb = 0, ja = 0, jb = 0;
#pragma unroll 1
    for (int b = wbits - 1; b >= 0; --b) {
        const u64 B = __ballot_sync(FULL, ina && ((Wa >> b) & 1)) | (u64(__ballot_sync(FULL, inb && ((Wb >> b) & 1))) << 32);
        if ((Wa >> b) & 1) {
            ja += __popcll(eqja & ~B);
            eqra &= B;
            eqja &= B;
        } else {
            ra += __popcll(eqra & B);
            eqra &= ~B;
            eqja &= ~B;
        }
        if ((Wb >> b) & 1) {
            jb += __popcll(eqjb & ~B);
            eqrb &= B;
            eqjb &= B;
        } else {
            rb += __popcll(eqrb & B);
            eqrb &= ~B;
            eqjb &= ~B;
        }
    }
    {
        const u64 lta = (1ull << va) - 1, ltb = (1ull << vb) - 1;  // equal W: smaller id first
        ra += __popcll(eqra & lta);
        ja += __popcll(eqja & lta);
        rb += __popcll(eqrb & ltb);
        jb += __popcll(eqjb & ltb);
    }
    // ---- block: the first join (in join order) v is an ancestor of, else the
    // residual (division.cpp:10-30) = arg-min of jpos over desc(v) ∩ J, one
    // jpos bit at a time (jpos < nj <= 63: six bits)
    const int nj = __popcll(J);
    int ba = 0, bb = 0;
    {
        u64 Ca = da & J, Cb = db & J;
#pragma unroll
        for (int b = 5; b >= 0; --b) {
            const u64 Z = __ballot_sync(FULL, ((J >> va) & 1) && !((ja >> b) & 1)) |
                          (u64(__ballot_sync(FULL, ((J >> vb) & 1) && !((jb >> b) & 1))) << 32);
            if (Ca & Z) Ca &= Z;
            else ba |= 1 << b;
            if (Cb & Z) Cb &= Z;
            else bb |= 1 << b;
        }
        if (!(da & J)) ba = nj;
        if (!(db & J)) bb = nj;
    }
    // ---- in-block depth = |anc(v) ∩ block(v)|: block member masks by shared
    // 64-bit atomics (S.pred is dead once pa / pb are in registers)
    unsigned long long* bmask = reinterpret_cast<unsigned long long*>(S.pred);
    bmask[lane] = 0;
    bmask[lane + 32] = 0;
    __syncwarp();
    if (ina) atomicOr(bmask + ba, 1ull << va);
    if (inb) atomicOr(bmask + bb, 1ull << vb);
    __syncwarp();
    const int dpa = ina ? __popcll(aa & bmask[ba]) : 0, dpb = inb ? __popcll(ab & bmask[bb]) : 0;
    // ---- division groups: (block, depth) in order; empty blocks vanish
    for (int i = lane; i < 68; i += 32) S.bdep[i] = 0;
    S.gcnt[lane] = 0;
    S.gcnt[lane + 32] = 0;
    S.gbig[lane] = 0;
    S.gbig[lane + 32] = 0;
    __syncwarp();
    if (ina) atomicMax(&S.bdep[ba], unsigned(dpa + 1));
    if (inb) atomicMax(&S.bdep[bb], unsigned(dpb + 1));
    __syncwarp();
    // exclusive prefix over blocks 0..nj (<= 65 entries, 3 per lane)
    u32 s0 = lane * 3 <= nj ? S.bdep[lane * 3] : 0u, s1 = lane * 3 + 1 <= nj ? S.bdep[lane * 3 + 1] : 0u,
        s2 = lane * 3 + 2 <= nj ? S.bdep[lane * 3 + 2] : 0u;
    u32 tot = s0 + s1 + s2, incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
    }
    const u32 ndiv = __shfl_sync(FULL, incl, 31);
    const u32 ex = incl - tot;
    __syncwarp();
    if (lane * 3 <= nj) S.bdep[lane * 3] = ex;
    if (lane * 3 + 1 <= nj) S.bdep[lane * 3 + 1] = ex + s0;
    if (lane * 3 + 2 <= nj) S.bdep[lane * 3 + 2] = ex + s0 + s1;
    __syncwarp();
    const int ga = ina ? int(S.bdep[ba]) + dpa : -1, gb = inb ? int(S.bdep[bb]) + dpb : -1;
    if (ina) {
        atomicAdd(&S.gcnt[ga], 1u);
        if (la >= u32(M)) S.gbig[ga] = 1;  // m^max = l >= M: oversized (division.cpp:99-101)
    }
    if (inb) {
        atomicAdd(&S.gcnt[gb], 1u);
        if (lb >= u32(M)) S.gbig[gb] = 1;
    }
    __syncwarp();
    // Rules 1-2 idle on every layer, else the general path
    const u32 ca = S.gcnt[lane], cb = S.gcnt[lane + 32];
    const bool cut = (ca > u32(M)) | (cb > u32(M)) | ((ca >= 2) & (S.gbig[lane] != 0)) |
                     ((cb >= 2) & (S.gbig[lane + 32] != 0));
    if (__any_sync(FULL, cut)) return -1;
    // ---- hand-off for k1_back_lane (K1Node, ro, divg, ndiv, shape key)
    if (ina) S.ord[ra] = (unsigned char)va;  // ranks are a permutation of 0..n-1
    if (inb) S.ord[rb] = (unsigned char)vb;
    __syncwarp();
    if (ina) {
        K1Node nd;
        nd.pred = pa;
        nd.ad = aa | da;
        nd.ln = la;
        nd.ld = 1;
        nd.pad = 0;
        a.h.node[n0 + va] = nd;
        a.h.ro[n0 + va] = uint16_t(ra | (S.ord[va] << 8));
    }
    if (inb) {
        K1Node nd;
        nd.pred = pb;
        nd.ad = ab | db;
        nd.ln = lb;
        nd.ld = 1;
        nd.pad = 0;
        a.h.node[n0 + vb] = nd;
        a.h.ro[n0 + vb] = uint16_t(rb | (S.ord[vb] << 8));
    }
    // division group member masks by shared 64-bit atomics (S.pred's block
    // masks are dead by now), then one coalesced store per group
    unsigned long long* gmask = reinterpret_cast<unsigned long long*>(S.pred);
    gmask[lane] = 0;
    gmask[lane + 32] = 0;
    __syncwarp();
    if (ina) atomicOr(gmask + ga, 1ull << va);
    if (inb) atomicOr(gmask + gb, 1ull << vb);
    __syncwarp();
    if (lane < int(ndiv)) a.h.divg[n0 + lane] = gmask[lane];
    if (lane + 32 < int(ndiv)) a.h.divg[n0 + lane + 32] = gmask[lane + 32];
    // walk-order key (walk_key): group count and member counts
    const u64 key = walk_key(lane, ndiv, lane < int(ndiv) ? ca : 0u, lane + 32 < int(ndiv) ? cb : 0u, false,
                             a.key_mode);
    if (lane == 0) {
        a.h.ndiv[d] = uint16_t(ndiv);
        a.status[d] = kStPending;
        if (a.h.skey) a.h.skey[d] = key;
    }
    return DS_OK;
}

// n <= 32 (86% of C5 DAGs): one node per lane, 32-bit masks, and each phase
// replaced by its cheapest warp form — W^anc by load bit-planes (popc of
// anc & plane), ranks and join positions by a bit-serial ballot count over
// the W^anc bits, blocks by a 5-step ballot arg-min over join positions,
// depth and division groups by __match_any_sync. ~700 warp instructions per
// DAG where the two-slot form (fast_dag) takes ~4000.
__device__ __forceinline__ int fast_dag32(FastWarp& S, const K1Args& a, const int lane, const u64 d, const u32 n0,
                                          const int n, const u32 e0, const int ne, const int M) {
    const bool in = lane < n;
    const u32 V = n == 32 ? FULL : ((1u << n) - 1);
    const u32 lt = (1u << lane) - 1;  // lanes below this one
    u32 l, p;
    if (a.tri.adj) {  // triangular wire form: u16 loads, predecessor bits
        l = in ? u32(a.tri.ln16[n0 + lane]) : 1u;
        if (__any_sync(FULL, l < 1)) return -1;
        const u32 w0 = a.tri.adj_off[d] - a.tri.adj_off[0], nw = a.tri.adj_off[d + 1] - a.tri.adj_off[d];
        p = u32(tri_preds(a.tri.adj + w0, nw, n, lane));
    } else {
        const long long l_ = in ? (long long)a.load_num[n0 + lane] : 1;
        if (__any_sync(FULL, l_ < 1 || l_ > 65535)) return -1;
        l = u32(l_);
        // ---- edges: every u < v < n (index order is topological), scattered to pred
        unsigned int* pr = reinterpret_cast<unsigned int*>(S.pred);
        pr[lane] = 0;
        __syncwarp();
        bool bad = false;
#pragma unroll 1
        for (int e = lane; e < ne; e += 32) {
            const u32 w = a.edges[e0 + e];
            const u32 u = w >> 16, v = w & 0xffffu;
            if (u >= v || v >= u32(n)) bad = true;
            else atomicOr(pr + v, 1u << u);
        }
        if (__any_sync(FULL, bad)) return -1;
        __syncwarp();
        p = in ? pr[lane] : 0u;
    }
    // ---- one source, one sink (dag.cpp:97-108)
    const u32 has_succ = __reduce_or_sync(FULL, p);
    if (__popc(__ballot_sync(FULL, in && p == 0)) != 1 || __popc(V & ~has_succ) != 1) return -1;
    // ---- closure, hop level, weighted prefix: one pass in index order
    const bool flat = !__any_sync(FULL, in && l > u32(M));
    const u32 w = l > u32(M) ? l : u32(M);  // exec(l, min(l, M)) in units of 1/M
    u32 an = 0, cpi = 0, pm = p;
    u32 rounds = 0;  // longest path in nodes
    if (flat) {
        // closure alone, one shuffle per node, over ancestors-or-self words x
        // (node k's word is shuffled as is; with k a compile-time constant
        // the predecessor test is one LOP3; one warp-uniform bound check per
        // 4 nodes — nodes >= n have x = 0 and no p bit). The longest path in
        // nodes by peeling sources layer by layer: v leaves in round lv(v) + 1
        u32 x = in ? (1u << lane) : 0u;
#pragma unroll
        for (int k0 = 0; k0 < 32; k0 += 4) {
            if (k0 >= n) break;
#pragma unroll
            for (int k = k0; k < k0 + 4; ++k) {
                const u32 ak = __shfl_sync(FULL, x, k);
                if ((p >> k) & 1) x |= ak;
            }
        }
        an = x & ~(1u << lane);
        for (u32 R = V; R; ++rounds) R &= ~__ballot_sync(FULL, ((R >> lane) & 1) && !(p & R));
    } else {
#pragma unroll 1
        for (int k = 0; k < n; ++k, pm >>= 1) {
            const u32 ak = __shfl_sync(FULL, an, k) | (1u << k);
            const u32 ck = __shfl_sync(FULL, cpi + w, k);
            if (pm & 1) {
                an |= ak;
                cpi = max(cpi, ck);
            }
        }
        for (u32 R = V; R; ++rounds) R &= ~__ballot_sync(FULL, ((R >> lane) & 1) && !(p & R));
    }
    const u32 de = warp_transpose32(an, lane);  // descendants (dag.cpp:119-124)
    // ---- bounds 1..4 (analysis.cpp:40-81)
    const u32 mask = a.mask;
    int64_t* bo = a.bounds + 10 * d;
    {
        const u32 U = __reduce_add_sync(FULL, in ? l : 0u);
        const u32 GU = flat ? u32(n) : __reduce_add_sync(FULL, in ? (l + u32(M) - 1) / u32(M) : 0u);
        const u32 G = flat ? u32(n) * u32(M) : __reduce_add_sync(FULL, in ? w : 0u);
        const u32 cp = flat ? rounds * u32(M) : __reduce_max_sync(FULL, in ? cpi + w : 0u);
        if (lane < 4) {  // greedy, greedy_unaware, graham_para, lower: one lane each
            const int k = lane + 1;
            u32 num = lane == 0 ? G : lane == 1 ? GU : lane == 2 ? rounds * u32(M) + U - rounds : (U > cp ? U : cp);
            u32 den = lane == 1 ? 1u : u32(M);
            const u32 g = gcd32(num, den);
            num /= g;
            den /= g;
            const bool want = mask & (1u << k);
            bo[2 * k] = want ? (long long)num : 0;
            bo[2 * k + 1] = want ? (long long)den : 0;
        }
    }
    if (!(mask & DS_M_PROPOSED)) {
        if (lane < 2) bo[lane] = 0;
        if (lane == 0) {
            a.status[d] = DS_OK;
            if (a.n_groups) a.n_groups[d] = 0;
            if (a.h.skey) a.h.skey[d] = kWalkKeyNone;
        }
        return DS_OK;
    }
    // ---- W^anc = l + sum over ancestors, by load bit-planes (dag.cpp:126-135)
    const int lbits = 32 - __clz(int(__reduce_or_sync(FULL, in ? l : 0u)));
    u32 W = l;
    // compile-time bit index (loads < 2^16), one bound check per 2 planes;
    // planes at or above lbits are empty and add nothing
#pragma unroll
    for (int b0 = 0; b0 < 16; b0 += 2) {
        if (b0 >= lbits) break;
#pragma unroll
        for (int b = b0; b < b0 + 2; ++b) W += u32(__popc(an & __ballot_sync(FULL, in && ((l >> b) & 1)))) << b;
    }
    // ---- rank (W desc, id asc) and join position (W asc, id asc), bit-serial
    const u32 J = __ballot_sync(FULL, in && __popc(p) >= 2);
    const int nj = __popc(J);
    const int wbits = 32 - __clz(int(__reduce_or_sync(FULL, in ? W : 0u)));
    u32 eqr = V, eqj = J;
    int rank = 0, jpos = 0;
#pragma unroll 1
    for (int b = wbits - 1; b >= 0; --b) {
        const u32 B = __ballot_sync(FULL, in && ((W >> b) & 1));
        if ((W >> b) & 1) {
            jpos += __popc(eqj & ~B);
            eqr &= B;
            eqj &= B;
        } else {
            rank += __popc(eqr & B);
            eqr &= ~B;
            eqj &= ~B;
        }
    }
    rank += __popc(eqr & lt);  // equal W: smaller id first
    jpos += __popc(eqj & lt);
    // ---- block: the first join (in join order) v is an ancestor of, else the
    // residual (division.cpp:10-30): arg-min of jpos over desc(v) ∩ J
    u32 C = de & J;
    int blk = 0;
#pragma unroll
    for (int b = 4; b >= 0; --b) {  // jpos < nj <= 31: five bits
        const u32 Z = __ballot_sync(FULL, ((J >> lane) & 1) && !((jpos >> b) & 1));
        if (C & Z) C &= Z;
        else blk |= 1 << b;
    }
    if (!(de & J)) blk = nj;
    // ---- in-block depth and division group (block, depth), in order
    const u32 bm = __match_any_sync(FULL, in ? blk : -1 - lane);
    const int dep = __popc(an & bm);
    S.bdep[lane] = 0;
    __syncwarp();
    if (in) atomicMax(&S.bdep[blk], unsigned(dep + 1));
    __syncwarp();
    const u32 layers = lane <= nj ? S.bdep[lane] : 0u;  // blocks 0..nj, one per lane (nj < 32)
    u32 incl = layers;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
    }
    const u32 ndiv = __shfl_sync(FULL, incl, 31);
    const int gidx = int(__shfl_sync(FULL, incl - layers, in ? blk : 0)) + dep;
    const u32 gm = __match_any_sync(FULL, in ? gidx : -1 - lane);
    const u32 cnt = __popc(gm);
    // Rules 1-2 idle on every layer, else the general path
    if (__any_sync(FULL, in && (cnt > u32(M) || (cnt >= 2 && l >= u32(M))))) return -1;
    // ---- compact hand-off for k1_back_lane (K1Rec16 run + u32 group masks in
    // the DAG's own slice of the K1Node array)
    K1Rec16* rec = reinterpret_cast<K1Rec16*>(a.h.node + n0);
    const bool leader = in && (gm & lt) == 0;
    if (leader) {
        reinterpret_cast<u32*>(rec + n)[gidx] = gm;
        S.gcnt[gidx] = cnt;
    }
    if (in) S.ord[rank] = (unsigned char)lane;
    __syncwarp();
    if (in) rec[lane] = K1Rec16{p, an | de, l, u32(rank) | (u32(S.ord[lane]) << 8)};
    const u64 key = walk_key(lane, ndiv, lane < int(ndiv) ? S.gcnt[lane] : 0u, 0u, true, a.key_mode);
    if (lane == 0) {
        a.h.ndiv[d] = uint16_t(ndiv) | kNdivCompact;
        a.status[d] = kStPending;
        if (a.h.skey) a.h.skey[d] = key;
    }
    return DS_OK;
}

// One warp per DAG. k1_fast<32> walks the whole batch, takes the DAGs with
// n <= 32 and lists those with 32 < n <= 64 for k1_fast<64> (h.l64); each
// queues what it cannot take for the general kernels (h.fb). Two kernels so
// each hot loop's code stays small (the SM's instruction cache).
template <int NMAX>
__global__ void __launch_bounds__(32 * kFastWarps) k1_fast(const K1Args a) {
    __shared__ FastWarp ws[kFastWarps];
    const int lane = threadIdx.x & 31;
    FastWarp& S = ws[threadIdx.x >> 5];
    const bool tri = a.tri.adj != nullptr;  // no edge list (widened later for the DAGs queued here)
    const u32 nbase = a.node_off[0], ebase = tri ? 0u : a.edge_off[0];
    const int M = a.plat.M;
    const u32 n_l64 = NMAX == 64 ? a.retry_count[kL64Counter] : 0u;
#pragma unroll 1
    for (;;) {
        u32 t = 0;
        if (lane == 0) t = atomicAdd(a.retry_count + (NMAX == 32 ? kFastCounter : kFast64Counter), 1u);
        t = __shfl_sync(FULL, t, 0);
        if (NMAX == 64 && t >= n_l64) break;
        const u64 d = NMAX == 64 ? a.h.l64[t] : t;
        if (d >= a.n_dags) break;
        const u32 n0 = a.node_off[d] - nbase, e0 = tri ? 0u : a.edge_off[d] - ebase;
        const int n = int(a.node_off[d + 1] - nbase - n0);
        const int ne = tri ? 0 : a.edge_cnt ? int(a.edge_cnt[d]) : int(a.edge_off[d + 1] - ebase - e0);
        int st;
        if (NMAX == 32) {
            if (n > 32 && n <= 64) {  // the two-slot kernel's
                if (lane == 0) a.h.l64[atomicAdd(a.retry_count + kL64Counter, 1u)] = u32(d);
                continue;
            }
            st = n >= 1 && n <= 32 ? fast_dag32(S, a, lane, d, n0, n, e0, ne, M) : -1;
        } else {
            st = fast_dag(S, a, lane, d, n0, n, e0, ne, M);
        }
        if (st != DS_OK && lane == 0) {
            a.h.fb[atomicAdd(a.retry_count + kFbCounter, 1u)] = u32(d);
            if (a.h.skey) a.h.skey[d] = kWalkKeyNone;  // not walked unless k1_mid takes it over
        }
        __syncwarp();
    }
}

// Walk order for k1_back_lane: within each window of kSortWindow consecutive
// DAGs (k1_mid / k1_fast put the window index in the key's high bits, so
// windows never mix), order the DAG indices by (shape key, index) — one CTA
// per window, a bitonic sort of 64-bit (key << 32 | index) words in shared
// memory (4096 x 8 B = 32 KB). Replaces a library radix sort; equal keys keep
// index order, as a stable sort would.
constexpr int kWsortThreads = 1024;
static_assert(kSortWindow == 4096, "k1_wsort sorts 4096-DAG windows");
// With `wcnt`, the window's walked DAGs are also counted by weight class, in
// sort order: wcnt[3w] light compact (key < heavy_key), wcnt[3w + 1] heavy
// compact (k1_fast<32> hand-offs with many division groups), wcnt[3w + 2]
// wide (K1Node hand-offs) — for k1_back_lane's heavy-first task order.
template <bool UNUSED = false>
__global__ void __launch_bounds__(kWsortThreads) k1_wsort(const u64* __restrict__ skey, u32* __restrict__ perm,
                                                           u64 n_dags, u32* __restrict__ wcnt, u64 heavy_key) {
    __shared__ u64 k[kSortWindow];
    const u64 base = u64(blockIdx.x) * kSortWindow;
    int c[3] = {0, 0, 0};
    for (int i = threadIdx.x; i < int(kSortWindow); i += kWsortThreads) {
        const u64 d = base + u64(i);
        const u64 key = d < n_dags ? skey[d] : kWalkKeyNone;
        k[i] = d < n_dags ? (key << 12) | u64(i) : ~0ull;  // 52-bit key, window-relative index
        if (key != kWalkKeyNone) ++c[((key >> 51) & 1) ? 2 : key >= heavy_key ? 1 : 0];
    }
    if (wcnt) {
        __shared__ int sc[3];
        if (threadIdx.x < 3) sc[threadIdx.x] = 0;
        __syncthreads();
        for (int j = 0; j < 3; ++j)
            if (c[j]) atomicAdd(&sc[j], c[j]);
        __syncthreads();
        if (threadIdx.x < 3) wcnt[3 * blockIdx.x + threadIdx.x] = u32(sc[threadIdx.x]);
    }
    __syncthreads();
#pragma unroll 1
    for (int size = 2; size <= int(kSortWindow); size <<= 1) {
#pragma unroll 1
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = threadIdx.x; t < int(kSortWindow) / 2; t += kWsortThreads) {
                const int lo = 2 * t - (t & (stride - 1)), hi = lo + stride;  // pair (lo, hi), lo's bit `stride` clear
                const bool up = (lo & size) == 0;
                const u64 x = k[lo], y = k[hi];
                if ((x > y) == up) {
                    k[lo] = y;
                    k[hi] = x;
                }
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < int(kSortWindow); i += kWsortThreads) {
        const u64 d = base + u64(i);
        if (d < n_dags) perm[d] = u32(base + (k[i] & 0xfffull));
    }
}

}  // namespace ds
