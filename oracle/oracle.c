/*
 * oracle.c — CPU oracle for batched sorted-array point lookups.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product path (paper_2506_01576_b200/, libbs.so) never links, imports or
 * calls it, and it shares no code, header, table or constant with the CUDA
 * path.
 *
 * What it computes (the plain definition, not a replay of the GPU algorithm):
 *
 *   lb(q)  = number of i in [0, n) with a[i] < q        (unsigned compare)
 *   hit(q) = lb(q) < n  and  a[lb(q)] == q
 *   out(q) = hit ? lb : (lb | MISS_BIT)                  MISS_BIT = top bit of
 *                                                        the output word
 *
 * Passages followed (PAPER.md line numbers, "P:n"):
 *   P:65  §3  "offset will point to the first entry not smaller than k"
 *             -> the answer is the textbook lower bound;
 *   P:69-81   Listing 1 — the same answer, clamped to n-1 on a miss above the
 *             maximum (reading R1/R3: results are reported as
 *             lb in [0, n] plus an explicit miss bit);
 *   pinning, reordering and K-ary search change
 *             only where the probes happen, never the per-query result.
 *   P:137 "rowID (or a miss)" -> explicit miss encoding (reading R3).
 *   P:61  "32-bit unsigned integers" -> unsigned compares everywhere (R20).
 *
 * Formulation: half-open bisection lo=0, hi=n; while lo<hi: mid=lo+(hi-lo)/2;
 * a[mid] < q ? lo=mid+1 : hi=mid.  Deliberately NOT the offset-based loop the
 * GPU kernels use.  Pinned against brute force, numpy.searchsorted, the
 * invariant a[lb-1] < q <= a[lb] and the paper's worked examples
 * (tests/test_oracle.py, tests/golden/).
 *
 * Standard-library free except <pthread.h> for the multi-threaded timing
 * driver (oracle_lookup_mt), which splits the queries into contiguous chunks.
 */
#include <pthread.h>

typedef unsigned long long u64;
typedef unsigned int u32;

/* ---------------- the definition ---------------- */

u64 oracle_lower_bound_u64(const u64* a, u64 n, u64 q) {
    u64 lo = 0, hi = n;
    while (lo < hi) {
        u64 mid = lo + (hi - lo) / 2;
        if (a[mid] < q) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

u64 oracle_lower_bound_u32(const u32* a, u64 n, u32 q) {
    u64 lo = 0, hi = n;
    while (lo < hi) {
        u64 mid = lo + (hi - lo) / 2;
        if (a[mid] < q) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

/* out word for one query.  key_bytes in {4, 8}; out_bytes in {4, 8}. */
static u64 oracle_encode(const void* keys, u64 n, int key_bytes, const void* q_ptr, u64 i,
                         int out_bytes) {
    u64 lb, hit;
    if (key_bytes == 8) {
        const u64* a = (const u64*)keys;
        u64 q = ((const u64*)q_ptr)[i];
        lb = oracle_lower_bound_u64(a, n, q);
        hit = (lb < n) && (a[lb] == q);
    } else {
        const u32* a = (const u32*)keys;
        u32 q = ((const u32*)q_ptr)[i];
        lb = oracle_lower_bound_u32(a, n, q);
        hit = (lb < n) && (a[lb] == q);
    }
    if (hit) return lb;
    if (out_bytes == 8) return lb | (1ull << 63);
    return lb | (1ull << 31);
}

/* Returns 0 on success, -1 on bad arguments. */
int oracle_lookup(const void* keys, u64 n, int key_bytes, const void* queries, u64 m,
                  void* out, int out_bytes) {
    u64 i;
    if ((key_bytes != 4 && key_bytes != 8) || (out_bytes != 4 && out_bytes != 8)) return -1;
    if (n == 0) return -1;
    if (out_bytes == 4 && n >= (1ull << 31)) return -1;
    for (i = 0; i < m; i++) {
        u64 r = oracle_encode(keys, n, key_bytes, queries, i, out_bytes);
        if (out_bytes == 8) ((u64*)out)[i] = r;
        else ((u32*)out)[i] = (u32)r;
    }
    return 0;
}

/* ---------------- multi-threaded driver (timing only) ---------------- */

typedef struct {
    const void* keys; u64 n; int key_bytes;
    const char* queries; u64 m; char* out; int out_bytes;
    int rc;
} oracle_job;

static void* oracle_worker(void* p) {
    oracle_job* j = (oracle_job*)p;
    j->rc = oracle_lookup(j->keys, j->n, j->key_bytes, j->queries, j->m, j->out, j->out_bytes);
    return 0;
}

/* Same result as oracle_lookup; queries split into `threads` contiguous chunks. */
int oracle_lookup_mt(const void* keys, u64 n, int key_bytes, const void* queries, u64 m,
                     void* out, int out_bytes, int threads) {
    enum { MAXT = 1024 };
    pthread_t tid[MAXT];
    int live[MAXT];
    oracle_job job[MAXT];
    int t, rc = 0;
    u64 per, off = 0;
    if (threads < 1) threads = 1;
    if (threads > MAXT) threads = MAXT;
    if ((u64)threads > m) threads = m ? (int)m : 1;
    per = (m + (u64)threads - 1) / (u64)threads;
    for (t = 0; t < threads; t++) {
        u64 c = (off + per <= m) ? per : (m - off);
        job[t].keys = keys; job[t].n = n; job[t].key_bytes = key_bytes;
        job[t].queries = (const char*)queries + off * (u64)key_bytes;
        job[t].m = c;
        job[t].out = (char*)out + off * (u64)out_bytes;
        job[t].out_bytes = out_bytes;
        job[t].rc = 0;
        off += c;
        live[t] = 0;
        if (t == 0) continue; /* chunk 0 runs on the calling thread */
        if (pthread_create(&tid[t], 0, oracle_worker, &job[t]) == 0) live[t] = 1;
        else oracle_worker(&job[t]);
    }
    oracle_worker(&job[0]);
    for (t = 1; t < threads; t++)
        if (live[t]) pthread_join(tid[t], 0);
    for (t = 0; t < threads; t++)
        if (job[t].rc) rc = job[t].rc;
    return rc;
}
