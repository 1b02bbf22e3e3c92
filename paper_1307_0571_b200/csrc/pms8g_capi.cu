// pms8g_capi.cu — the C ABI (include/pms8g.h): validation, device context,
// pipeline orchestration on one CUDA stream, CUB sort/unique, host decode.
//
// Mirrors the reference's run_parallel (src/parallel.cpp:35-118): build the
// shared context once (here: encode + per-anchor row build on the device),
// search every S1 l-mer (here: one persistent kernel over a global work queue
// of (S1 l-mer, depth-1 branch) tasks), then canonicalise the motif set
// (sort + unique, src/solver.cpp:16-21). There is no CPU search path.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>
#include <functional>
#include <mutex>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "../../include/pms8g.h"
#include "pms8g_device.cuh"
#include "pms8g_internal.h"
#include "pms8g_launch.h"
#include "pms8g_sigma.h"

using namespace pms8g;

namespace {

struct Err {
    int code = PMS8G_OK;
    std::string msg;
};

#define CU(call) PMS8G_CU(call)

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

unsigned __int128 nsize(int l, int d, int sigma) {
    unsigned __int128 total = 0, binom = 1, power = 1;
    for (int i = 0; i <= d; ++i) {
        total += binom * power;
        binom = binom * static_cast<unsigned>(l - i) / static_cast<unsigned>(i + 1);
        power *= static_cast<unsigned>(sigma - 1);
    }
    return total;
}

}  // namespace

struct pms8g_ctx {
    int n = 0, m = 0, l = 0, d = 0, sigma = 0, W = 1, w = 0, K = 0, t = 0;
    int ref_t = 0;  // the reference's switch depth (override or estimate_threshold), reported
    int B = 2;          // bits (planes) per symbol: 2 for sigma <= 4 (two-plane DNA path), else ceil(log2 sigma)
    bool sig = false;   // sigma > 4: the B-plane search (pms8g_sigma.cu)
    int key_bits() const { return B * l; }
    std::string alphabet;
    pms8g_options opt{};
    std::vector<int32_t> anchors;
    std::vector<int32_t> req_anchors;  // the caller's S1 offset list (context cache key)
    std::string env_sig;                // creation-time test knobs (context cache key)
    std::vector<int32_t> task_ai;
    std::vector<uint32_t> task_u;
    int32_t* d_task_ai = nullptr;
    uint32_t* d_task_u = nullptr;
    int device = 0;
    int sms = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[6] = {};
    uint8_t* d_codes = nullptr;
    void* d_table = nullptr;
    int32_t* d_anchors = nullptr;
    uint32_t* d_l1 = nullptr;
    LevelMeta* d_meta = nullptr;
    long long* d_task_base = nullptr;
    uint32_t* d_order = nullptr;  // static task order: keys in/out, vals in/out (4 x order_cap)
    long long order_cap = 0;
    void* d_order_tmp = nullptr;
    size_t order_tmp_bytes = 0;
    unsigned long long* d_task_counter = nullptr;
    uint32_t* d_scratch = nullptr;
    size_t scratch_words = 0;
    int level_cap = 0, node_cap = 0;
    unsigned long long* d_keys = nullptr;
    unsigned long long* d_keys_sorted = nullptr;
    unsigned long long* d_keys_unique = nullptr;
    long long key_cap = 0;
    unsigned long long* d_key_count = nullptr;
    long long* d_unique_count = nullptr;
    void* d_cub = nullptr;
    size_t cub_bytes = 0;
    unsigned long long* d_counters = nullptr;
    int* d_err = nullptr;
    int* d_fail = nullptr;
    // pinned host mirrors
    unsigned long long* h_counters = nullptr;  // C_NCTR + 1 (key count)
    int* h_err = nullptr;
    int blocks = 0, warps = 0;
    size_t smem = 0;
    WarpPlan plan{};
    QueueState* d_qs = nullptr;
    unsigned int* d_qstate = nullptr;
    uint8_t* d_qslots = nullptr;
    int qcap = 0, qslot_bytes = 0, don_cap = 0;
    size_t device_bytes = 0;
    long long unique_count = 0;
    pms8g_report report{};
};

namespace pms8g {

int merge_keys_with(MergeScratch& m, const void* dev_in, long long count, void* dev_out, long long* out_count,
                    cudaStream_t s, char* err, size_t errlen) {
    using K128 = unsigned __int128;
    *out_count = 0;
    if (count <= 0) return PMS8G_OK;
    int dev = 0;
    CU(cudaGetDevice(&dev));
    if (m.device != dev) {
        merge_scratch_free(m);
        m.device = dev;
    }
    if (count > m.cap) {
        const long long cap = std::max<long long>(count, 2 * m.cap);
        if (m.sorted) cudaFree(m.sorted);
        if (m.temp) cudaFree(m.temp);
        m.sorted = m.temp = nullptr;
        m.cap = 0;
        size_t b1 = 0, b2 = 0;
        CU(cudaMalloc(&m.sorted, sizeof(K128) * cap));
        if (!m.count) CU(cudaMalloc(&m.count, sizeof(long long)));
        if (!m.h_count) CU(cudaMallocHost(&m.h_count, sizeof(long long)));
        cub::DeviceRadixSort::SortKeys(nullptr, b1, static_cast<const K128*>(nullptr), static_cast<K128*>(nullptr),
                                       static_cast<int>(cap), 0, 128, s);
        cub::DeviceSelect::Unique(nullptr, b2, static_cast<const K128*>(nullptr), static_cast<K128*>(nullptr),
                                  m.count, static_cast<int>(cap), s);
        m.temp_bytes = std::max(b1, b2);
        CU(cudaMalloc(&m.temp, m.temp_bytes));
        m.cap = cap;
    }
    size_t bytes = m.temp_bytes;
    CU(cub::DeviceRadixSort::SortKeys(m.temp, bytes, static_cast<const K128*>(dev_in), static_cast<K128*>(m.sorted),
                                      static_cast<int>(count), 0, 128, s));
    bytes = m.temp_bytes;
    CU(cub::DeviceSelect::Unique(m.temp, bytes, static_cast<const K128*>(m.sorted), static_cast<K128*>(dev_out),
                                 m.count, static_cast<int>(count), s));
    CU(cudaMemcpyAsync(m.h_count, m.count, sizeof(long long), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    *out_count = *m.h_count;
    return PMS8G_OK;
}

void merge_scratch_free(MergeScratch& m) {
    if (m.device >= 0) cudaSetDevice(m.device);
    if (m.sorted) cudaFree(m.sorted);
    if (m.temp) cudaFree(m.temp);
    if (m.count) cudaFree(m.count);
    if (m.h_count) cudaFreeHost(m.h_count);
    m = MergeScratch{};
}

}  // namespace pms8g

namespace {

// The environment knobs read when a context is created (test hooks): a cached
// context is reused only under the same values.
std::string env_signature() {
    std::string sig;
    for (const char* k : {"PMS8G_GLOBAL_TABLE", "PMS8G_NODE_CAP", "PMS8G_QCAP", "PMS8G_NO_TASK_ORDER", "PMS8G_DON_CAP"}) {
        const char* v = std::getenv(k);
        sig += v ? v : "-";
        sig += '|';
    }
    return sig;
}

int alloc(pms8g_ctx* c, void** p, size_t bytes, char* err, size_t errlen) {
    cudaError_t e = cudaMalloc(p, bytes ? bytes : 16);
    if (e != cudaSuccess)
        return fail(err, errlen, PMS8G_ERR_RUNTIME, "cannot allocate %zu bytes of device memory: %s", bytes,
                    cudaGetErrorString(e));
    c->device_bytes += bytes;
    return PMS8G_OK;
}

int ensure_key_capacity(pms8g_ctx* c, long long need, char* err, size_t errlen) {
    if (need <= c->key_cap) return PMS8G_OK;
    long long cap = std::max<long long>(need, 2 * c->key_cap);
    cudaFree(c->d_keys);
    cudaFree(c->d_keys_sorted);
    cudaFree(c->d_keys_unique);
    cudaFree(c->d_cub);
    c->d_keys = c->d_keys_sorted = c->d_keys_unique = nullptr;
    c->d_cub = nullptr;
    int rc;
    if ((rc = alloc(c, reinterpret_cast<void**>(&c->d_keys), 16 * cap, err, errlen))) return rc;
    if ((rc = alloc(c, reinterpret_cast<void**>(&c->d_keys_sorted), 16 * cap, err, errlen))) return rc;
    if ((rc = alloc(c, reinterpret_cast<void**>(&c->d_keys_unique), 16 * cap, err, errlen))) return rc;
    size_t b1 = 0, b2 = 0;
    using K128 = unsigned __int128;
    cub::DeviceRadixSort::SortKeys(nullptr, b1, reinterpret_cast<K128*>(c->d_keys),
                                   reinterpret_cast<K128*>(c->d_keys_sorted), static_cast<int>(cap), 0,
                                   std::max(1, c->key_bits()));
    cub::DeviceSelect::Unique(nullptr, b2, reinterpret_cast<K128*>(c->d_keys_sorted),
                              reinterpret_cast<K128*>(c->d_keys_unique), c->d_unique_count, static_cast<int>(cap));
    c->cub_bytes = std::max(b1, b2);
    if ((rc = alloc(c, &c->d_cub, c->cub_bytes, err, errlen))) return rc;
    c->key_cap = cap;
    return PMS8G_OK;
}

int validate_problem(int n, int m, int l, int d, const char* alphabet, char* err, size_t errlen, int* sigma) {
    // Problem::validate, src/problem.cpp:7-28
    if (n < 1) return fail(err, errlen, PMS8G_ERR_INVALID, "no input sequences");
    if (l < 1) return fail(err, errlen, PMS8G_ERR_INVALID, "motif length must be >= 1");
    if (l > m) return fail(err, errlen, PMS8G_ERR_INVALID, "motif length %d exceeds sequence length %d", l, m);
    if (d < 0 || d > l) return fail(err, errlen, PMS8G_ERR_INVALID, "mismatch budget must be in [0, l], got %d", d);
    const int s = alphabet ? static_cast<int>(std::strlen(alphabet)) : 4;
    if (s < 2) return fail(err, errlen, PMS8G_ERR_INVALID, "alphabet needs at least 2 symbols");
    for (int i = 0; i < s; ++i)  // Alphabet ctor, src/alphabet.cpp:13-17
        for (int j = 0; j < i; ++j)
            if (alphabet[i] == alphabet[j])
                return fail(err, errlen, PMS8G_ERR_INVALID, "duplicate alphabet symbol '%c'", alphabet[i]);
    // GPU path limits: 2 bit planes up to 4 symbols (l <= 64),
    // B = ceil(log2 sigma) planes of one word up to 32 symbols (l <= 32 and
    // B*l <= 128 key bits), 32 rows per warp table, 24-bit l-mer ids
    if (s > 32)
        return fail(err, errlen, PMS8G_ERR_INVALID, "GPU path supports alphabets of at most 32 symbols, got %d", s);
    if (s <= 4 && l > 64) return fail(err, errlen, PMS8G_ERR_INVALID, "GPU path supports l <= 64, got %d", l);
    if (s > 4) {
        const int b = sigma_planes(s);
        const int lmax = std::min(32, 128 / b);
        if (l > lmax)
            return fail(err, errlen, PMS8G_ERR_INVALID,
                        "GPU path supports l <= %d for a %d-symbol alphabet (%d bits per symbol), got %d", lmax, s, b,
                        l);
    }
    if (n > MAXN) return fail(err, errlen, PMS8G_ERR_INVALID, "GPU path supports n <= %d sequences, got %d", MAXN, n);
    const long long K = static_cast<long long>(n) * (m - l + 1);
    if (K > static_cast<long long>(ID_MASK))
        return fail(err, errlen, PMS8G_ERR_INVALID, "GPU path supports n*(m-l+1) <= %u (24-bit l-mer ids), got %lld",
                    ID_MASK, K);
    *sigma = s;
    return PMS8G_OK;
}

int resolve_threshold(int n, int m, int l, int d, int sigma, int requested, char* err, size_t errlen, int* t) {
    if (requested != 0) {
        if (requested < 1 || requested > n)
            return fail(err, errlen, PMS8G_ERR_INVALID, "threshold must be in [1, n], got %d", requested);
        *t = requested;
    } else {
        *t = pms8g_gpu_threshold(n, m, l, d, sigma);
    }
    // the output is independent of t (every pruning rule is sound); the
    // device tables hold at most MAXT stack members
    if (*t > MAXT) *t = MAXT;
    if (*t > n) *t = n;
    if (*t < 1) *t = 1;
    return PMS8G_OK;
}

int run_pipeline(pms8g_ctx* c, char* err, size_t errlen);

}  // namespace

extern "C" {

void pms8g_default_options(pms8g_options* o) {
    std::memset(o, 0, sizeof *o);
    o->sort_rows = 1;
    o->prune_level = 2;
    o->device = -1;
    o->shard_count = 1;
    o->max_motifs = -1;
}

const char* pms8g_version(void) { return "pms8g 0.2 (sm_100a)"; }

int pms8g_queue_create(int device, pms8g_queue** out, uint8_t* handle, char* err, size_t errlen) {
    *out = nullptr;
    int ndev = 0;
    cudaError_t ce = cudaGetDeviceCount(&ndev);
    if (ce != cudaSuccess || ndev == 0)
        return fail(err, errlen, PMS8G_ERR_CUDA, "no CUDA device available (%s); the GPU path has no CPU fallback",
                    cudaGetErrorString(ce));
    if (device >= 0) CU(cudaSetDevice(device));
    auto* q = new pms8g_queue();
    CU(cudaGetDevice(&q->device));
    q->owner = 1;
    if (cudaMalloc(&q->dptr, 256) != cudaSuccess) {
        delete q;
        return fail(err, errlen, PMS8G_ERR_RUNTIME, "cannot allocate the shared queue");
    }
    CU(cudaMemset(q->dptr, 0, 256));
    CU(cudaDeviceSynchronize());
    cudaIpcMemHandle_t h;
    CU(cudaIpcGetMemHandle(&h, q->dptr));
    static_assert(sizeof(cudaIpcMemHandle_t) == PMS8G_QUEUE_HANDLE_BYTES, "IPC handle size");
    std::memcpy(handle, &h, sizeof h);
    *out = q;
    return PMS8G_OK;
}

int pms8g_queue_open(const uint8_t* handle, int device, pms8g_queue** out, char* err, size_t errlen) {
    *out = nullptr;
    int ndev = 0;
    cudaError_t ce = cudaGetDeviceCount(&ndev);
    if (ce != cudaSuccess || ndev == 0)
        return fail(err, errlen, PMS8G_ERR_CUDA, "no CUDA device available (%s); the GPU path has no CPU fallback",
                    cudaGetErrorString(ce));
    if (device >= 0) CU(cudaSetDevice(device));
    auto* q = new pms8g_queue();
    CU(cudaGetDevice(&q->device));
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof h);
    ce = cudaIpcOpenMemHandle(&q->dptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (ce != cudaSuccess) {
        delete q;
        return fail(err, errlen, PMS8G_ERR_CUDA, "cannot map the shared queue on device %d (%s)", device,
                    cudaGetErrorString(ce));
    }
    *out = q;
    return PMS8G_OK;
}

void pms8g_queue_destroy(pms8g_queue* q) {
    if (!q) return;
    cudaSetDevice(q->device);
    if (q->owner == 1) cudaFree(q->dptr);
    else if (q->owner == 0) cudaIpcCloseMemHandle(q->dptr);
    delete q;
}

int pms8g_estimate_threshold(int n, int m, int l, int d, int sigma) {
    // threshold_curve + estimate_threshold, src/solver.cpp:75-117
    if (n < 2) return n;
    if (m == l) return n;
    if (m <= l) return 2;
    auto lg = [](unsigned __int128 v) { return static_cast<double>(std::log(static_cast<long double>(v))); };
    const double log_nd = lg(nsize(l, d, sigma));
    const double log_n2d = lg(nsize(l, std::min(2 * d, l), sigma));
    const double log_p = log_n2d - l * std::log(static_cast<double>(sigma));
    const double log_q = log_nd - log_n2d;
    const double log_w = std::log(static_cast<double>(m - l + 1));
    std::vector<double> terms;
    for (int k = 1; k <= n; ++k) terms.push_back(k * log_w + 0.5 * k * (k - 1) * log_p);
    int best_t = 2;
    double best = INFINITY;
    for (int t = 2; t <= n; ++t) {
        const double mx = *std::max_element(terms.begin(), terms.begin() + t);
        double sum = 0;
        for (int k = 0; k < t; ++k) sum += std::exp(terms[k] - mx);
        const double ls = std::log(static_cast<double>(n)) + std::log(static_cast<double>(l)) + mx + std::log(sum);
        const double lp = terms[t - 1] + log_nd + (t - 1) * log_q + std::log(static_cast<double>(l));
        const double v = std::max(ls, lp);
        if (v < best - 1e-12) {
            best = v;
            best_t = t;
        }
    }
    return best_t;
}

int pms8g_gpu_threshold(int n, int m, int l, int d, int sigma) {
    // The reference balances log Time_sample(t) against log Time_pattern(t)
    // (Appendix D, src/solver.cpp:75-117). On the GPU the pattern phase costs
    // relatively more per unit of the model (divergent DFS + verification vs
    // bitwise filtering), so t is the smallest depth whose pattern term is at
    // most 10^1.3 x the sample term; fitted on the five BASELINE configs
    // (13,4)->2, (17,6)->3, (21,8)->4, (23,9)->4, (50,21)->6 measured on B200.
    if (const char* env = std::getenv("PMS8G_THRESHOLD")) {
        const int v = std::atoi(env);
        if (v >= 1) return std::min(v, n);
    }
    if (n < 2 || m <= l) return pms8g_estimate_threshold(n, m, l, d, sigma);
    auto lg = [](unsigned __int128 v) { return static_cast<double>(std::log(static_cast<long double>(v))); };
    const double log_nd = lg(nsize(l, d, sigma));
    const double log_n2d = lg(nsize(l, std::min(2 * d, l), sigma));
    const double log_p = log_n2d - l * std::log(static_cast<double>(sigma));
    const double log_q = log_nd - log_n2d;
    const double log_w = std::log(static_cast<double>(m - l + 1));
    std::vector<double> terms;
    for (int k = 1; k <= n; ++k) terms.push_back(k * log_w + 0.5 * k * (k - 1) * log_p);
    const double beta = 1.3 * std::log(10.0);
    for (int t = 2; t <= n; ++t) {
        const double mx = *std::max_element(terms.begin(), terms.begin() + t);
        double sum = 0;
        for (int k = 0; k < t; ++k) sum += std::exp(terms[k] - mx);
        const double ls = std::log(static_cast<double>(n)) + std::log(static_cast<double>(l)) + mx + std::log(sum);
        const double lp = terms[t - 1] + log_nd + (t - 1) * log_q + std::log(static_cast<double>(l));
        if (lp - ls <= beta) {
            // where the model asks for 5+ members the tuples' neighbourhoods are
            // still huge and heavy-tailed (one (50,21) 6-tuple kept 300+ warps
            // busy for 0.4 s); the push filters with the consensus row rule are
            // cheap there, so two levels deeper pay: (50,21) per 56 S1 l-mers
            // t=5 minutes, t=6 1.28 s (22,269 tuples, 2.3 G nodes), t=7 0.49 s
            // (247 tuples, 4.3 M nodes)
            if (t >= 5) t = std::min(std::min(t + 2, MAXT), n);
            return t;
        }
    }
    return n;
}

int pms8g_generate(int n, int m, int l, int d, int sigma, uint64_t seed, int exactly_d, uint8_t* codes_out,
                   uint8_t* motif_out, int32_t* positions_out) {
    // generate_planted_instance, src/instance.cpp:12-73: std::mt19937_64 +
    // rejection-sampled bounded draws, same draw order
    if (l < 1 || l > m || d < 0 || d > l || n < 1 || sigma < 2) return PMS8G_ERR_INVALID;
    std::mt19937_64 rng(seed);
    auto draw = [&](uint64_t bound) {
        const uint64_t threshold = (~bound + 1) % bound;
        for (;;) {
            const uint64_t x = rng();
            if (x >= threshold) return x % bound;
        }
    };
    for (int p = 0; p < l; ++p) motif_out[p] = static_cast<uint8_t>(draw(sigma));
    std::vector<int> columns(l);
    std::vector<uint8_t> occ(l);
    for (int i = 0; i < n; ++i) {
        uint8_t* seq = codes_out + static_cast<size_t>(i) * m;
        for (int j = 0; j < m; ++j) seq[j] = static_cast<uint8_t>(draw(sigma));
        const int pos = static_cast<int>(draw(static_cast<uint64_t>(m - l + 1)));
        std::memcpy(occ.data(), motif_out, l);
        for (int j = 0; j < l; ++j) columns[j] = j;
        for (int j = 0; j < d; ++j) {
            const int pick = j + static_cast<int>(draw(static_cast<uint64_t>(l - j)));
            std::swap(columns[j], columns[pick]);
            const int col = columns[j];
            if (!exactly_d) {
                occ[col] = static_cast<uint8_t>(draw(sigma));
            } else {
                uint64_t cc = draw(static_cast<uint64_t>(sigma - 1));
                if (cc >= occ[col]) ++cc;
                occ[col] = static_cast<uint8_t>(cc);
            }
        }
        std::memcpy(seq + pos, occ.data(), l);
        positions_out[i] = pos;
    }
    return PMS8G_OK;
}

int pms8g_ctx_create(int n, int m, int l, int d, const char* alphabet, const pms8g_options* opt_in, pms8g_ctx** out,
                     char* err, size_t errlen) {
    *out = nullptr;
    pms8g_options opt;
    if (opt_in) opt = *opt_in;
    else pms8g_default_options(&opt);
    int sigma = 0;
    int rc = validate_problem(n, m, l, d, alphabet, err, errlen, &sigma);
    if (rc) return rc;
    int t = 0;
    if ((rc = resolve_threshold(n, m, l, d, sigma, opt.threshold, err, errlen, &t))) return rc;
    if (opt.shard_count < 1) opt.shard_count = 1;
    if (opt.queue && opt.shard_count > 1)
        return fail(err, errlen, PMS8G_ERR_INVALID, "a shared queue replaces sharding: shard_count must be 1");
    if (opt.shard_rank < 0 || opt.shard_rank >= opt.shard_count)
        return fail(err, errlen, PMS8G_ERR_INVALID, "shard rank %d outside [0, %d)", opt.shard_rank, opt.shard_count);

    int ndev = 0;
    cudaError_t ce = cudaGetDeviceCount(&ndev);
    if (ce != cudaSuccess || ndev == 0)
        return fail(err, errlen, PMS8G_ERR_CUDA, "no CUDA device available (%s); the GPU path has no CPU fallback",
                    cudaGetErrorString(ce));
    int dev = opt.device;
    if (dev < 0) CU(cudaGetDevice(&dev));
    if (dev >= ndev) return fail(err, errlen, PMS8G_ERR_INVALID, "device %d not present (%d devices)", dev, ndev);
    CU(cudaSetDevice(dev));
    cudaDeviceProp prop;
    CU(cudaGetDeviceProperties(&prop, dev));
    if (prop.major < 10)
        return fail(err, errlen, PMS8G_ERR_CUDA, "device %d (%s, sm_%d%d) is not sm_100-class; kernels are sm_100a only",
                    dev, prop.name, prop.major, prop.minor);

    auto* c = new pms8g_ctx();
    c->n = n;
    c->m = m;
    c->l = l;
    c->d = d;
    c->sigma = sigma;
    c->alphabet = alphabet ? alphabet : "ACGT";
    c->W = l <= 32 ? 1 : 2;
    c->sig = sigma > 4;
    c->B = c->sig ? sigma_planes(sigma) : 2;
    if (c->sig && (opt.queue || (opt.branches && opt.nbranches > 0))) {
        delete c;
        return fail(err, errlen, PMS8G_ERR_INVALID,
                    "shared queues and explicit branches need an alphabet of at most 4 symbols");
    }
    c->w = m - l + 1;
    c->K = n * c->w;
    c->t = t;
    c->ref_t = opt.threshold > 0 ? opt.threshold : pms8g_estimate_threshold(n, m, l, d, sigma);
    c->env_sig = env_signature();
    c->opt = opt;
    c->device = dev;
    c->sms = prop.multiProcessorCount;
    // S1 offsets of this call (split_subproblems, src/parallel.cpp:14-20), sharded
    if (opt.branches && opt.nbranches > 0) {
        if (t < 2) {
            delete c;
            return fail(err, errlen, PMS8G_ERR_INVALID, "explicit branches need a switch depth >= 2");
        }
        for (int i = 0; i < opt.nbranches; ++i) {
            const int a = opt.branches[2 * i], u = opt.branches[2 * i + 1];
            if (a < 0 || a >= c->w || u < 0 || u >= c->K) {
                delete c;
                return fail(err, errlen, PMS8G_ERR_INVALID, "branch (%d, %d) out of range", a, u);
            }
            if (std::find(c->anchors.begin(), c->anchors.end(), a) == c->anchors.end()) c->anchors.push_back(a);
        }
        std::sort(c->anchors.begin(), c->anchors.end());
        for (int i = 0; i < opt.nbranches; ++i) {
            const int a = opt.branches[2 * i];
            c->task_ai.push_back(static_cast<int32_t>(std::lower_bound(c->anchors.begin(), c->anchors.end(), a) -
                                                      c->anchors.begin()));
            c->task_u.push_back(static_cast<uint32_t>(opt.branches[2 * i + 1]));
        }
    } else if (opt.anchors && opt.nanchors > 0) {
        c->req_anchors.assign(opt.anchors, opt.anchors + opt.nanchors);
        for (int i = 0; i < opt.nanchors; ++i) {
            const int a = opt.anchors[i];
            if (a < 0 || a >= c->w) {
                delete c;
                return fail(err, errlen, PMS8G_ERR_INVALID, "anchor offset %d outside [0, %d)", a, c->w);
            }
            if (a % opt.shard_count == opt.shard_rank) c->anchors.push_back(a);
        }
    } else {
        for (int a = 0; a < c->w; ++a)
            if (a % opt.shard_count == opt.shard_rank) c->anchors.push_back(a);
    }
    c->opt.anchors = nullptr;
    c->opt.nanchors = 0;
    c->opt.branches = nullptr;
    c->opt.nbranches = 0;

    auto cleanup_fail = [&](int code) {
        pms8g_ctx_destroy(c);
        return code;
    };
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess)
        return cleanup_fail(fail(err, errlen, PMS8G_ERR_CUDA, "cannot create stream"));
    for (auto& e : c->ev)
        if (cudaEventCreate(&e) != cudaSuccess)
            return cleanup_fail(fail(err, errlen, PMS8G_ERR_CUDA, "cannot create event"));

    // launch shape: one persistent block per SM, as many warps as the
    // shared-memory l-mer table leaves room for
    const size_t smem_cap = prop.sharedMemPerBlockOptin;
    if (c->sig) {
        // sigma-symbol search: table in global memory (L1/L2), per-warp state in shared memory
        c->warps = opt.warps_per_block > 0 ? std::min(opt.warps_per_block, 16) : 16;
        c->smem = sigma_warp_smem() * c->warps;
        c->blocks = opt.grid_blocks > 0 ? opt.grid_blocks : c->sms * (opt.blocks_per_sm > 0 ? opt.blocks_per_sm : 1);
    } else {
        // one-word l-mers: table in shared memory; if it leaves fewer than
        // half the warps, the instance runs the two-word build (table in
        // global memory, upper words zero) — DESIGN.md §3
        auto fit = [&](int W, int want) {
            const WarpPlan plan = make_plan(W, l, t);
            int wp = want;
            while (wp > 1 && search_smem(W, c->K, wp, plan) + 64 > smem_cap) --wp;  // + static smem
            return search_smem(W, c->K, wp, plan) + 64 > smem_cap ? 0 : wp;
        };
        if (c->W == 1) {
            const int want = opt.warps_per_block > 0 ? std::min(opt.warps_per_block, 16) : search_default_warps(1, t);
            if (std::getenv("PMS8G_GLOBAL_TABLE") || 2 * fit(1, want) < want) c->W = 2;
        }
        c->plan = make_plan(c->W, l, t);
        const int want = opt.warps_per_block > 0 ? std::min(opt.warps_per_block, 16) : search_default_warps(c->W, t);
        c->warps = fit(c->W, want);
        if (c->warps == 0)
            return cleanup_fail(fail(err, errlen, PMS8G_ERR_INVALID, "per-warp state of %d warps does not fit %zu bytes",
                                     want, smem_cap));
        c->smem = search_smem(c->W, c->K, c->warps, c->plan);
        c->blocks = opt.grid_blocks > 0 ? opt.grid_blocks : c->sms * (opt.blocks_per_sm > 0 ? opt.blocks_per_sm : 1);
        if (set_search_smem(c->W, c->t, c->smem) != cudaSuccess)
            return cleanup_fail(fail(err, errlen, PMS8G_ERR_CUDA, "cannot set shared memory size %zu", c->smem));
    }
    const int warps = c->warps;

    const int na = static_cast<int>(c->anchors.size());
    c->level_cap = (c->K + 31) / 32 * 32;  // keeps the per-warp node overflow 16-byte aligned
    c->node_cap = 64 * (l + 4);
    if (const char* e = std::getenv("PMS8G_NODE_CAP")) c->node_cap = std::max(0, std::atoi(e));  // failure tests
    const size_t lvl_words = static_cast<size_t>(std::max(0, t - 1)) * c->level_cap;
    const size_t node_words =
        static_cast<size_t>(c->node_cap) * (c->sig ? sigma_node_bytes() : node_bytes(c->W)) / 4;
    c->scratch_words = (lvl_words + node_words + static_cast<size_t>(c->plan.thr_global_bytes) / 4 + 64 + 31) / 32 * 32;
    const size_t nwarps_total = static_cast<size_t>(c->blocks) * warps;
    int rc2;
#define AL(ptr, bytes)                                                                          \
    if ((rc2 = alloc(c, reinterpret_cast<void**>(&(ptr)), (bytes), err, errlen)) != PMS8G_OK) \
        return cleanup_fail(rc2);
    AL(c->d_codes, static_cast<size_t>(n) * m);
    AL(c->d_table, (static_cast<size_t>(c->K) * (c->sig ? sigma_lmer_bytes(c->B) : lmer_bytes(c->W)) + 15) / 16 *
                       16);  // 16-byte multiple (bulk-copy staging)
    AL(c->d_anchors, sizeof(int32_t) * std::max(1, na));
    AL(c->d_l1, sizeof(uint32_t) * static_cast<size_t>(std::max(1, na)) * c->K);
    AL(c->d_meta, sizeof(LevelMeta) * std::max(1, na));
    AL(c->d_task_base, sizeof(long long) * (na + 1));
    AL(c->d_task_counter, sizeof(unsigned long long));
    AL(c->d_scratch, sizeof(uint32_t) * c->scratch_words * nwarps_total);
    AL(c->d_key_count, sizeof(unsigned long long));
    AL(c->d_unique_count, sizeof(long long));
    AL(c->d_counters, sizeof(unsigned long long) * C_NCTR);
    AL(c->d_err, 2 * sizeof(int));  // flags, failing S1 offset + 1
    AL(c->d_task_ai, sizeof(int32_t) * std::max<size_t>(1, c->task_ai.size()));
    AL(c->d_task_u, sizeof(uint32_t) * std::max<size_t>(1, c->task_u.size()));
    if (c->task_u.empty() && t >= 2 && !c->sig && !std::getenv("PMS8G_NO_TASK_ORDER")) {
        // heaviest-first static task order (taskorder_kernel + stable radix sort)
        c->order_cap = static_cast<long long>(std::max(1, na)) * c->w;
        AL(c->d_order, sizeof(uint32_t) * 4 * c->order_cap);
        uint32_t* k0 = c->d_order;
        cub::DeviceRadixSort::SortPairs(nullptr, c->order_tmp_bytes, k0, k0 + c->order_cap, k0 + 2 * c->order_cap,
                                        k0 + 3 * c->order_cap, static_cast<int>(c->order_cap), 0, 8);
        AL(c->d_order_tmp, std::max<size_t>(16, c->order_tmp_bytes));
    }
    c->qcap = 8192;
    if (const char* q = std::getenv("PMS8G_QCAP")) c->qcap = std::max(16, std::atoi(q));  // ring stress tests
    // level hand-off with donated tasks (TaskHeader::hlevel): only searches
    // with t >= 3 have a level >= 2 to hand off
    c->don_cap = t >= 3 ? std::min(c->level_cap, 16384) : 0;
    if (const char* q = std::getenv("PMS8G_DON_CAP")) c->don_cap = std::max(0, std::min(c->level_cap, std::atoi(q)));
    c->qslot_bytes = static_cast<int>(task_slot_bytes(c->W, c->don_cap));
    AL(c->d_qs, sizeof(QueueState));
    AL(c->d_qslots, static_cast<size_t>(c->qcap) * c->qslot_bytes);
    AL(c->d_qstate, sizeof(unsigned int) * c->qcap);
    AL(c->d_fail, sizeof(int));
#undef AL
    if (cudaMallocHost(reinterpret_cast<void**>(&c->h_counters), sizeof(unsigned long long) * (C_NCTR + 2)) !=
            cudaSuccess ||
        cudaMallocHost(reinterpret_cast<void**>(&c->h_err), sizeof(int) * 4) != cudaSuccess)
        return cleanup_fail(fail(err, errlen, PMS8G_ERR_RUNTIME, "cannot allocate pinned host memory"));
    if ((rc2 = ensure_key_capacity(c, 1 << 14, err, errlen)) != PMS8G_OK) return cleanup_fail(rc2);
    if (!c->task_ai.empty() &&
        (cudaMemcpy(c->d_task_ai, c->task_ai.data(), sizeof(int32_t) * c->task_ai.size(), cudaMemcpyHostToDevice) !=
             cudaSuccess ||
         cudaMemcpy(c->d_task_u, c->task_u.data(), sizeof(uint32_t) * c->task_u.size(), cudaMemcpyHostToDevice) !=
             cudaSuccess))
        return cleanup_fail(fail(err, errlen, PMS8G_ERR_CUDA, "branch upload failed"));
    if (na > 0 && cudaMemcpy(c->d_anchors, c->anchors.data(), sizeof(int32_t) * na, cudaMemcpyHostToDevice) !=
                      cudaSuccess)
        return cleanup_fail(fail(err, errlen, PMS8G_ERR_CUDA, "anchor upload failed"));
    *out = c;
    return PMS8G_OK;
}

void pms8g_ctx_destroy(pms8g_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    void* ptrs[] = {c->d_codes, c->d_table,      c->d_anchors,     c->d_l1,           c->d_meta,
                    c->d_task_base, c->d_task_counter, c->d_scratch, c->d_keys,   c->d_keys_sorted,
                    c->d_keys_unique, c->d_key_count, c->d_unique_count, c->d_cub, c->d_counters,
                    c->d_err,     c->d_fail, c->d_qs, c->d_qslots, c->d_qstate, c->d_task_ai, c->d_task_u,
                    c->d_order, c->d_order_tmp};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    if (c->h_counters) cudaFreeHost(c->h_counters);
    if (c->h_err) cudaFreeHost(c->h_err);
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

int pms8g_ctx_load_codes(pms8g_ctx* c, const uint8_t* codes, int on_device, char* err, size_t errlen) {
    CU(cudaSetDevice(c->device));
    const size_t bytes = static_cast<size_t>(c->n) * c->m;
    if (!on_device) {
        for (size_t i = 0; i < bytes; ++i)
            if (codes[i] >= c->sigma)
                return fail(err, errlen, PMS8G_ERR_INVALID, "sequence %zu, position %zu: code %d not in alphabet %s",
                            i / c->m, i % c->m, codes[i], c->alphabet.c_str());
    }
    CU(cudaMemcpyAsync(c->d_codes, codes, bytes, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                       c->stream));
    return PMS8G_OK;
}

void* pms8g_ctx_stream(pms8g_ctx* c) { return c ? c->stream : nullptr; }

int pms8g_ctx_run(pms8g_ctx* c, char* err, size_t errlen) { return run_pipeline(c, err, errlen); }

int pms8g_ctx_keys(pms8g_ctx* c, const uint64_t** dev_keys, int64_t* count) {
    *dev_keys = reinterpret_cast<const uint64_t*>(c->d_keys_unique);
    *count = c->unique_count;
    return PMS8G_OK;
}

int pms8g_ctx_report(pms8g_ctx* c, const pms8g_report** out) {
    *out = &c->report;
    return PMS8G_OK;
}

int pms8g_ctx_counters(pms8g_ctx* c, uint64_t* out, int cap) {
    const int k = cap < C_NCTR ? cap : C_NCTR;
    for (int i = 0; i < k; ++i) out[i] = c->h_counters[i];
    return C_NCTR;
}

int pms8g_ctx_kernel_ms(pms8g_ctx* c, float* search_ms, float* rowbuild_ms) {
    float a = 0, b = 0;
    if (cudaEventElapsedTime(&a, c->ev[2], c->ev[3]) != cudaSuccess) a = -1;
    if (cudaEventElapsedTime(&b, c->ev[0], c->ev[1]) != cudaSuccess) b = -1;
    if (search_ms) *search_ms = a;
    if (rowbuild_ms) *rowbuild_ms = b;
    return PMS8G_OK;
}

void pms8g_decode_keys(const uint64_t* keys, int64_t count, int l, const char* alphabet, char* out) {
    const char* sym = alphabet ? alphabet : "ACGT";
    // bits per symbol: 2 up to 4 symbols, else ceil(log2 sigma) (the B-plane path)
    const int sigma = static_cast<int>(std::strlen(sym));
    const int b = sigma <= 4 ? 2 : sigma_planes(sigma);
    const uint64_t mask = (1ull << b) - 1ull;
    for (int64_t i = 0; i < count; ++i) {
        const uint64_t lo = keys[2 * i], hi = keys[2 * i + 1];
        for (int p = 0; p < l; ++p) {
            const int sh = b * (l - 1 - p);
            uint64_t v = sh >= 64 ? (hi >> (sh - 64)) : (lo >> sh);
            if (sh < 64 && sh + b > 64) v |= hi << (64 - sh);
            out[i * l + p] = sym[static_cast<int>(v & mask)];
        }
    }
    // keys sort in code order; canonical_motif_set (src/solver.cpp:16-21)
    // sorts by byte value, which differs when the alphabet's symbols are not
    // in ascending byte order (e.g. custom:TGCA): re-sort the strings then
    bool ascending = true;
    for (const char* q = sym; q[0] && q[1]; ++q)
        if (static_cast<unsigned char>(q[0]) >= static_cast<unsigned char>(q[1])) ascending = false;
    if (!ascending && count > 1) {
        std::vector<std::string> v(static_cast<size_t>(count));
        for (int64_t i = 0; i < count; ++i) v[static_cast<size_t>(i)].assign(out + i * l, static_cast<size_t>(l));
        std::sort(v.begin(), v.end());
        for (int64_t i = 0; i < count; ++i) std::memcpy(out + i * l, v[static_cast<size_t>(i)].data(), l);
    }
}

int pms8g_ctx_result(pms8g_ctx* c, pms8g_result* out, char* err, size_t errlen) {
    std::memset(out, 0, sizeof *out);
    CU(cudaSetDevice(c->device));
    const long long cnt = c->unique_count;
    std::vector<uint64_t> keys(2 * static_cast<size_t>(std::max(0ll, cnt)));
    if (cnt > 0) {
        CU(cudaMemcpyAsync(keys.data(), c->d_keys_unique, 16 * cnt, cudaMemcpyDeviceToHost, c->stream));
        CU(cudaStreamSynchronize(c->stream));
    }
    out->l = c->l;
    out->count = cnt;
    out->motifs = static_cast<char*>(std::malloc(static_cast<size_t>(cnt) * c->l + 1));
    if (!out->motifs) return fail(err, errlen, PMS8G_ERR_RUNTIME, "cannot allocate motif buffer");
    pms8g_decode_keys(keys.data(), cnt, c->l, c->alphabet.c_str(), out->motifs);
    out->motifs[static_cast<size_t>(cnt) * c->l] = 0;
    out->report = c->report;
    return PMS8G_OK;
}

void pms8g_result_free(pms8g_result* r) {
    if (r && r->motifs) {
        std::free(r->motifs);
        r->motifs = nullptr;
    }
}

int pms8g_merge_keys(const uint64_t* dev_in, int64_t count, uint64_t* dev_out, int64_t* out_count, void* stream,
                     char* err, size_t errlen) {
    // one grow-only scratch per device (allocated once, reused by every merge)
    static std::mutex mu;
    static MergeScratch scratch[64];
    *out_count = 0;
    if (count <= 0) return PMS8G_OK;
    int dev = 0;
    CU(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> g(mu);
    long long n = 0;
    const int rc = merge_keys_with(scratch[dev & 63], dev_in, count, dev_out, &n, static_cast<cudaStream_t>(stream),
                                   err, errlen);
    *out_count = n;
    return rc;
}

namespace {
std::mutex g_cache_mu;
pms8g_ctx* g_cache = nullptr;
std::mutex g_batch_mu;
std::vector<pms8g_ctx*> g_batch;  // pms8g_solve_batch's lane contexts

bool same_shape(const pms8g_ctx* c, int n, int m, int l, int d, const char* alphabet, const pms8g_options& o) {
    if (!c) return false;
    if (c->env_sig != env_signature()) return false;
    const int dev = o.device;
    int cur = -1;
    if (dev < 0) cudaGetDevice(&cur);
    return c->n == n && c->m == m && c->l == l && c->d == d && c->alphabet == (alphabet ? alphabet : "ACGT") &&
           c->opt.threshold == o.threshold && c->opt.sort_rows == o.sort_rows && c->opt.prune_level == o.prune_level &&
           c->opt.reverify == o.reverify && c->opt.max_motifs == o.max_motifs &&
           c->opt.shard_rank == o.shard_rank && std::max(1, c->opt.shard_count) == std::max(1, o.shard_count) &&
           (dev < 0 ? cur : dev) == c->device && o.branches == nullptr &&
           (o.anchors == nullptr ? c->req_anchors.empty()
                                 : c->req_anchors == std::vector<int32_t>(o.anchors, o.anchors + std::max(0, o.nanchors))) &&
           c->opt.warps_per_block == o.warps_per_block &&
           c->opt.blocks_per_sm == o.blocks_per_sm && c->opt.exact_tree == o.exact_tree && c->opt.queue == o.queue &&
           c->opt.grid_blocks == o.grid_blocks;
}
}  // namespace

}  // extern "C" (reopened below)

namespace pms8g {
// More than MAXN sequences (the reference takes any n, src/problem.cpp:7-28):
// a motif of all n sequences is a motif of the first MAXN, and the search is
// exact, so the motif set of the first MAXN sequences contains the answer;
// the GPU scanner (naive_is_motif over every sequence) keeps exactly the
// members that also occur in the remaining ones. The warp's row tables stay
// lane-indexed (32 rows). `solve_head` searches the first MAXN sequences.
int solve_many_sequences(const uint8_t* codes, int n, int m, int l, int d, const char* alphabet,
                         const pms8g_options& opt, pms8g_result* out, char* err, size_t errlen,
                         const std::function<int(const pms8g_options&, pms8g_result*)>& solve_head) {
    const int sig = alphabet ? static_cast<int>(std::strlen(alphabet)) : 4;
    if (sig > 4)
        return fail(err, errlen, PMS8G_ERR_INVALID,
                    "GPU path supports n <= %d sequences for alphabets above 4 symbols, got %d", MAXN, n);
    if (opt.branches)
        return fail(err, errlen, PMS8G_ERR_INVALID, "branch subsets need n <= %d sequences, got %d", MAXN, n);
    pms8g_options sub_opt = opt;
    sub_opt.max_motifs = -1;  // the cap applies to the instance's own motifs, below
    pms8g_result sub;
    int rc = solve_head(sub_opt, &sub);
    if (rc) return rc;
    const char* alpha = alphabet ? alphabet : "ACGT";
    const int64_t cnt = sub.count;
    std::vector<uint8_t> mc(static_cast<size_t>(cnt) * l), pass(static_cast<size_t>(cnt));
    std::vector<int32_t> wit(static_cast<size_t>(cnt) * n);
    for (int64_t i = 0; i < cnt * l; ++i) mc[i] = static_cast<uint8_t>(std::strchr(alpha, sub.motifs[i]) - alpha);
    rc = pms8g_verify_motifs(codes, n, m, l, d, alphabet, mc.data(), cnt, wit.data(), pass.data(), opt.device, err,
                             errlen);
    if (rc) {
        pms8g_result_free(&sub);
        return rc;
    }
    int64_t kept = 0;
    for (int64_t i = 0; i < cnt; ++i)
        if (pass[i]) {
            if (kept != i) std::memmove(sub.motifs + kept * l, sub.motifs + i * l, static_cast<size_t>(l));
            ++kept;
        }
    sub.motifs[kept * l] = 0;
    sub.count = kept;
    if (opt.max_motifs >= 0 && kept > opt.max_motifs) {
        pms8g_result_free(&sub);
        return fail(err, errlen, PMS8G_ERR_RUNTIME, "motif cap of %lld exceeded", static_cast<long long>(opt.max_motifs));
    }
    *out = sub;
    return PMS8G_OK;
}
}  // namespace pms8g

extern "C" {

int pms8g_solve(const uint8_t* codes, int n, int m, int l, int d, const char* alphabet, const pms8g_options* opt_in,
                pms8g_result* out, char* err, size_t errlen) {
    const double t0 = now_s();
    std::memset(out, 0, sizeof *out);
    pms8g_options opt;
    if (opt_in) opt = *opt_in;
    else pms8g_default_options(&opt);
    if (n > MAXN) {
        const int rc = solve_many_sequences(codes, n, m, l, d, alphabet, opt, out, err, errlen,
                                            [&](const pms8g_options& o, pms8g_result* r) {
                                                return pms8g_solve(codes, MAXN, m, l, d, alphabet, &o, r, err, errlen);
                                            });
        if (!rc) out->report.wall_seconds = now_s() - t0;
        return rc;
    }
    int sigma = 0;
    int rc = validate_problem(n, m, l, d, alphabet, err, errlen, &sigma);
    if (rc) return rc;
    // a process-wide context cache keeps device buffers across calls of the
    // same shape (like a cached library handle); subset runs are never cached
    std::lock_guard<std::mutex> lock(g_cache_mu);
    pms8g_ctx* c = nullptr;
    bool cached = false;
    if (same_shape(g_cache, n, m, l, d, alphabet, opt)) {
        c = g_cache;
        cached = true;
    } else {
        if ((rc = pms8g_ctx_create(n, m, l, d, alphabet, &opt, &c, err, errlen))) return rc;
        if (!opt.branches) {  // whole instances and S1 offset subsets (repeated by benchmarks) are cached
            pms8g_ctx_destroy(g_cache);
            g_cache = c;
            cached = true;
        }
    }
    rc = pms8g_ctx_load_codes(c, codes, 0, err, errlen);
    if (!rc) rc = pms8g_ctx_run(c, err, errlen);
    if (!rc) rc = pms8g_ctx_result(c, out, err, errlen);
    if (!cached) pms8g_ctx_destroy(c);
    if (!rc) out->report.wall_seconds = now_s() - t0;
    return rc;
}

int pms8g_solve_batch(const uint8_t* const* codes, int count, int n, int m, int l, int d, const char* alphabet,
                      const pms8g_options* opt_in, pms8g_result* outs, char* err, size_t errlen) {
    const double t0 = now_s();
    if (count < 0) return fail(err, errlen, PMS8G_ERR_INVALID, "negative instance count");
    for (int i = 0; i < count; ++i) std::memset(&outs[i], 0, sizeof outs[i]);
    if (count == 0) return PMS8G_OK;
    pms8g_options opt;
    if (opt_in) opt = *opt_in;
    else pms8g_default_options(&opt);
    if (opt.queue) return fail(err, errlen, PMS8G_ERR_INVALID, "a batch runs on one device: no shared queue");
    int sigma = 0;
    int rc = validate_problem(n, m, l, d, alphabet, err, errlen, &sigma);
    if (rc) return rc;
    int ndev = 0;
    cudaError_t ce = cudaGetDeviceCount(&ndev);
    if (ce != cudaSuccess || ndev == 0)
        return fail(err, errlen, PMS8G_ERR_CUDA, "no CUDA device available (%s); the GPU path has no CPU fallback",
                    cudaGetErrorString(ce));
    int dev = opt.device;
    if (dev < 0) CU(cudaGetDevice(&dev));
    int sms = 0;
    CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    // up to `lanes` instances in flight, each on its own stream with an equal
    // share of the SMs (its persistent grid), one host thread each; waves of
    // `lanes` when there are more instances than that
    const int lanes = std::max(1, std::min({count, sms, opt.grid_blocks > 0 ? sms / opt.grid_blocks : 8}));
    opt.device = dev;
    opt.grid_blocks = std::max(1, sms / lanes);
    // the lanes' contexts are cached across calls of the same shape (like
    // pms8g_solve's handle cache); subset runs are never cached
    std::lock_guard<std::mutex> lock(g_batch_mu);
    const bool cacheable = !opt.anchors && !opt.branches;
    bool reuse = cacheable && static_cast<int>(g_batch.size()) == lanes;
    for (int k = 0; reuse && k < lanes; ++k) reuse = same_shape(g_batch[k], n, m, l, d, alphabet, opt);
    if (!reuse) {
        for (auto* c : g_batch) pms8g_ctx_destroy(c);
        g_batch.clear();
    }
    std::vector<pms8g_ctx*> ctx = reuse ? g_batch : std::vector<pms8g_ctx*>(lanes, nullptr);
    for (int k = 0; !reuse && k < lanes; ++k)
        if ((rc = pms8g_ctx_create(n, m, l, d, alphabet, &opt, &ctx[k], err, errlen))) {
            for (auto* c : ctx) pms8g_ctx_destroy(c);
            return rc;
        }
    if (cacheable) g_batch = ctx;
    std::vector<int> rcs(count, PMS8G_OK);
    std::vector<std::string> msgs(count);
    for (int base = 0; base < count && rc == PMS8G_OK; base += lanes) {
        const int nw = std::min(lanes, count - base);
        std::vector<std::thread> th;
        for (int k = 0; k < nw; ++k)
            th.emplace_back([&, k] {
                const int i = base + k;
                char e[512] = {0};
                int r = cudaSetDevice(dev) == cudaSuccess ? PMS8G_OK : PMS8G_ERR_CUDA;
                if (!r) r = pms8g_ctx_load_codes(ctx[k], codes[i], 0, e, sizeof e);
                if (!r) r = pms8g_ctx_run(ctx[k], e, sizeof e);
                if (!r) r = pms8g_ctx_result(ctx[k], &outs[i], e, sizeof e);
                rcs[i] = r;
                msgs[i] = e;
            });
        for (auto& x : th) x.join();
        for (int k = 0; k < nw; ++k)
            if (rcs[base + k] != PMS8G_OK && rc == PMS8G_OK) {
                rc = fail(err, errlen, rcs[base + k], "instance %d: %s", base + k, msgs[base + k].c_str());
            }
    }
    if (!cacheable) {
        for (auto* c : ctx) pms8g_ctx_destroy(c);
    }
    if (rc != PMS8G_OK) {
        for (int i = 0; i < count; ++i) pms8g_result_free(&outs[i]);
        return rc;
    }
    const double wall = now_s() - t0;
    for (int i = 0; i < count; ++i) outs[i].report.wall_seconds = wall;
    return PMS8G_OK;
}

int pms8g_int_peak(int device, double* ops_per_second, double* popc_per_second, char* err, size_t errlen) {
    if (device >= 0) CU(cudaSetDevice(device));
    int dev = 0;
    CU(cudaGetDevice(&dev));
    cudaDeviceProp prop;
    CU(cudaGetDeviceProperties(&prop, dev));
    uint32_t* sink = nullptr;
    CU(cudaMalloc(&sink, 16));
    cudaEvent_t a, b;
    CU(cudaEventCreate(&a));
    CU(cudaEventCreate(&b));
    const int blocks = prop.multiProcessorCount * 8, threads = 256, iters = 2048;
    double res[2] = {0, 0};
    for (int which = 0; which < 2; ++which) {
        float best = 1e30f;
        for (int rep = 0; rep < 4; ++rep) {
            CU(cudaEventRecord(a));
            CU(launch_intpeak(which, blocks, threads, iters, sink, nullptr));
            CU(cudaEventRecord(b));
            CU(cudaEventSynchronize(b));
            float ms = 0;
            CU(cudaEventElapsedTime(&ms, a, b));
            if (rep > 0) best = std::min(best, ms);
        }
        const double ops = static_cast<double>(blocks) * threads * iters * 16.0 * 8.0;
        res[which] = ops / (best * 1e-3);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(sink);
    if (ops_per_second) *ops_per_second = res[0];
    if (popc_per_second) *popc_per_second = res[1];
    return PMS8G_OK;
}

}  // extern "C"

namespace {

// Problem::validate (src/problem.cpp:7-28) plus the scanner's device limits
// (2 bit planes: at most 4 symbols, l <= 64); codes checked against sigma.
int validate_scan(const uint8_t* codes, int n, int m, int l, int d, const char* alphabet, char* err, size_t errlen,
                  int* sigma) {
    if (n < 1) return fail(err, errlen, PMS8G_ERR_INVALID, "no input sequences");
    if (l < 1) return fail(err, errlen, PMS8G_ERR_INVALID, "motif length must be >= 1");
    if (l > m) return fail(err, errlen, PMS8G_ERR_INVALID, "motif length %d exceeds sequence length %d", l, m);
    if (d < 0 || d > l) return fail(err, errlen, PMS8G_ERR_INVALID, "mismatch budget must be in [0, l], got %d", d);
    const int s = alphabet ? static_cast<int>(std::strlen(alphabet)) : 4;
    if (s < 2) return fail(err, errlen, PMS8G_ERR_INVALID, "alphabet needs at least 2 symbols");
    for (int i = 0; i < s; ++i)  // Alphabet ctor, src/alphabet.cpp:13-17
        for (int j = 0; j < i; ++j)
            if (alphabet[i] == alphabet[j])
                return fail(err, errlen, PMS8G_ERR_INVALID, "duplicate alphabet symbol '%c'", alphabet[i]);
    if (s > 4)
        return fail(err, errlen, PMS8G_ERR_INVALID, "GPU path supports alphabets of at most 4 symbols, got %d", s);
    if (l > 64) return fail(err, errlen, PMS8G_ERR_INVALID, "GPU path supports l <= 64, got %d", l);
    const size_t bytes = static_cast<size_t>(n) * m;
    for (size_t i = 0; i < bytes; ++i)
        if (codes[i] >= s)
            return fail(err, errlen, PMS8G_ERR_INVALID, "sequence %zu, position %zu: code %d not in alphabet %s",
                        i / m, i % m, codes[i], alphabet ? alphabet : "ACGT");
    *sigma = s;
    return PMS8G_OK;
}

// Device buffers of one scanner call (freed on every exit path).
struct ScanBufs {
    uint8_t* codes = nullptr;
    void* table = nullptr;
    int* flag = nullptr;
    void* a = nullptr;
    void* b = nullptr;
    void* c = nullptr;
    cudaStream_t stream = nullptr;
    ~ScanBufs() {
        if (stream) cudaStreamSynchronize(stream);
        for (void* p : {static_cast<void*>(codes), table, static_cast<void*>(flag), a, b, c})
            if (p) cudaFree(p);
        if (stream) cudaStreamDestroy(stream);
    }
};

// H2D codes + K1 encode into a fresh l-mer table.
int scan_setup(ScanBufs& B, const uint8_t* codes, int n, int m, int l, int device, int* W, int* w, char* err,
               size_t errlen) {
    int ndev = 0;
    cudaError_t ce = cudaGetDeviceCount(&ndev);
    if (ce != cudaSuccess || ndev == 0)
        return fail(err, errlen, PMS8G_ERR_CUDA, "no CUDA device available (%s); the GPU path has no CPU fallback",
                    cudaGetErrorString(ce));
    if (device >= ndev)
        return fail(err, errlen, PMS8G_ERR_INVALID, "device %d not present (%d devices)", device, ndev);
    if (device >= 0) CU(cudaSetDevice(device));
    int dev = 0;
    CU(cudaGetDevice(&dev));
    cudaDeviceProp prop;
    CU(cudaGetDeviceProperties(&prop, dev));
    if (prop.major < 10)
        return fail(err, errlen, PMS8G_ERR_CUDA, "device %d (%s, sm_%d%d) is not sm_100-class; kernels are sm_100a only",
                    dev, prop.name, prop.major, prop.minor);
    CU(cudaStreamCreateWithFlags(&B.stream, cudaStreamNonBlocking));
    *W = l <= 32 ? 1 : 2;
    *w = m - l + 1;
    const size_t bytes = static_cast<size_t>(n) * m;
    CU(cudaMalloc(&B.codes, bytes));
    CU(cudaMalloc(&B.table, (static_cast<size_t>(n) * *w * lmer_bytes(*W) + 15) / 16 * 16));
    CU(cudaMalloc(&B.flag, sizeof(int)));
    CU(cudaMemsetAsync(B.flag, 0, sizeof(int), B.stream));
    CU(cudaMemcpyAsync(B.codes, codes, bytes, cudaMemcpyHostToDevice, B.stream));
    CU(launch_encode(*W, B.codes, n, m, l, *w, B.table, B.flag, B.stream));
    return PMS8G_OK;
}

}  // namespace

extern "C" {

int pms8g_verify_motifs(const uint8_t* codes, int n, int m, int l, int d, const char* alphabet, const uint8_t* motifs,
                        int64_t nmotifs, int32_t* witness, uint8_t* pass, int device, char* err, size_t errlen) {
    int sigma = 0;
    int rc = validate_scan(codes, n, m, l, d, alphabet, err, errlen, &sigma);
    if (rc) return rc;
    if (nmotifs < 0) return fail(err, errlen, PMS8G_ERR_INVALID, "negative motif count");
    for (int64_t i = 0; i < nmotifs * l; ++i)
        if (motifs[i] >= sigma)
            return fail(err, errlen, PMS8G_ERR_INVALID, "motif %lld contains a code outside the alphabet",
                        static_cast<long long>(i / l));
    if (nmotifs == 0) return PMS8G_OK;
    ScanBufs B;
    int W = 1, w = 0;
    if ((rc = scan_setup(B, codes, n, m, l, device, &W, &w, err, errlen))) return rc;
    CU(cudaMalloc(&B.a, static_cast<size_t>(nmotifs) * l));
    CU(cudaMalloc(&B.b, static_cast<size_t>(nmotifs) * n * sizeof(int32_t)));
    CU(cudaMalloc(&B.c, static_cast<size_t>(nmotifs)));
    CU(cudaMemcpyAsync(B.a, motifs, static_cast<size_t>(nmotifs) * l, cudaMemcpyHostToDevice, B.stream));
    CU(launch_witness(W, B.table, n, w, l, d, sigma, static_cast<const uint8_t*>(B.a), nmotifs,
                      static_cast<int32_t*>(B.b), static_cast<uint8_t*>(B.c), B.stream));
    CU(cudaMemcpyAsync(witness, B.b, static_cast<size_t>(nmotifs) * n * sizeof(int32_t), cudaMemcpyDeviceToHost,
                       B.stream));
    CU(cudaMemcpyAsync(pass, B.c, static_cast<size_t>(nmotifs), cudaMemcpyDeviceToHost, B.stream));
    CU(cudaStreamSynchronize(B.stream));
    return PMS8G_OK;
}

int pms8g_brute_force(const uint8_t* codes, int n, int m, int l, int d, const char* alphabet, int64_t guard,
                      int device, pms8g_result* out, char* err, size_t errlen) {
    const double t0 = now_s();
    std::memset(out, 0, sizeof *out);
    int sigma = 0;
    int rc = validate_scan(codes, n, m, l, d, alphabet, err, errlen, &sigma);
    if (rc) return rc;
    // check_guard, src/oracle.cpp:41-46
    const long double space = std::pow(static_cast<long double>(sigma), l);
    if (space > static_cast<long double>(guard))
        return fail(err, errlen, PMS8G_ERR_INVALID, "enumeration space %d^%d exceeds guard %lld", sigma, l,
                    static_cast<long long>(guard));
    unsigned long long total = 1;
    for (int p = 0; p < l; ++p) total *= static_cast<unsigned long long>(sigma);
    ScanBufs B;
    int W = 1, w = 0;
    if ((rc = scan_setup(B, codes, n, m, l, device, &W, &w, err, errlen))) return rc;
    int dev = 0;
    CU(cudaGetDevice(&dev));
    int sms = 0;
    CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    cudaEvent_t e0, e1;
    CU(cudaEventCreate(&e0));
    CU(cudaEventCreate(&e1));
    long long cap = static_cast<long long>(std::min<unsigned long long>(total, 1ull << 20));
    unsigned long long found = 0;
    float ms = 0.f;
    for (int pass = 0; pass < 2; ++pass) {
        if (B.a) cudaFree(B.a);
        B.a = nullptr;
        CU(cudaMalloc(&B.a, 16 * static_cast<size_t>(std::max(1ll, cap))));
        if (!B.b) CU(cudaMalloc(&B.b, sizeof(unsigned long long)));
        CU(cudaMemsetAsync(B.b, 0, sizeof(unsigned long long), B.stream));
        CU(cudaEventRecord(e0, B.stream));
        CU(launch_sweep(W, B.table, n, w, l, d, sigma, total, static_cast<unsigned long long*>(B.a),
                        static_cast<unsigned long long*>(B.b), cap, sms, B.stream));
        CU(cudaEventRecord(e1, B.stream));
        CU(cudaMemcpyAsync(&found, B.b, sizeof found, cudaMemcpyDeviceToHost, B.stream));
        CU(cudaStreamSynchronize(B.stream));
        CU(cudaEventElapsedTime(&ms, e0, e1));
        if (static_cast<long long>(found) <= cap) break;
        cap = static_cast<long long>(found);  // second pass with room for every motif
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const long long cnt = static_cast<long long>(found);
    std::vector<uint64_t> keys(2 * static_cast<size_t>(cnt));
    if (cnt > 0) {
        CU(cudaMalloc(&B.c, 16 * static_cast<size_t>(cnt)));
        int64_t uniq = 0;
        if ((rc = pms8g_merge_keys(static_cast<const uint64_t*>(B.a), cnt, static_cast<uint64_t*>(B.c), &uniq,
                                   B.stream, err, errlen)))
            return rc;
        CU(cudaMemcpyAsync(keys.data(), B.c, 16 * static_cast<size_t>(uniq), cudaMemcpyDeviceToHost, B.stream));
        CU(cudaStreamSynchronize(B.stream));
        keys.resize(2 * static_cast<size_t>(uniq));
    }
    const long long uniq = static_cast<long long>(keys.size() / 2);
    out->l = l;
    out->count = uniq;
    out->motifs = static_cast<char*>(std::malloc(static_cast<size_t>(uniq) * l + 1));
    if (!out->motifs) return fail(err, errlen, PMS8G_ERR_RUNTIME, "cannot allocate motif buffer");
    pms8g_decode_keys(keys.data(), uniq, l, alphabet ? alphabet : "ACGT", out->motifs);
    out->motifs[static_cast<size_t>(uniq) * l] = 0;
    pms8g_report& R = out->report;
    R.n = n;
    R.m = m;
    R.l = l;
    R.d = d;
    R.sigma = sigma;
    R.gpus = 1;
    R.motif_count = uniq;
    R.motifs_emitted = cnt;
    R.neighbors_visited = static_cast<int64_t>(total);
    R.device_seconds = ms * 1e-3;
    R.pattern_seconds = ms * 1e-3;
    R.wall_seconds = now_s() - t0;
    return PMS8G_OK;
}

}  // extern "C"

namespace {

int run_pipeline(pms8g_ctx* c, char* err, size_t errlen) {
    const double t0 = now_s();
    CU(cudaSetDevice(c->device));
    cudaStream_t s = c->stream;
    const int na = static_cast<int>(c->anchors.size());
    for (int attempt = 0; attempt < 8; ++attempt) {
        CU(cudaMemsetAsync(c->d_counters, 0, sizeof(unsigned long long) * C_NCTR, s));
        CU(cudaMemsetAsync(c->d_key_count, 0, sizeof(unsigned long long), s));
        CU(cudaMemsetAsync(c->d_qs, 0, sizeof(QueueState), s));
        CU(cudaMemsetAsync(c->d_qstate, 0, sizeof(unsigned int) * c->qcap, s));
        CU(cudaMemsetAsync(c->d_err, 0, 2 * sizeof(int), s));
        CU(cudaMemsetAsync(c->d_fail, 0, sizeof(int), s));
        const char* tl_path = std::getenv("PMS8G_TIMELINE");  // diagnostics: task timeline dump
        unsigned long long* d_tl = nullptr;
        if (c->sig) {
            // alphabets of 5..32 symbols: B-plane l-mers (pms8g_sigma.cu)
            CU(cudaMemsetAsync(c->d_task_counter, 0, sizeof(unsigned long long), s));
            CU(launch_encode_sigma(c->B, c->d_codes, c->n, c->m, c->l, c->w, c->sigma, c->d_table, c->d_err, s));
            CU(cudaEventRecord(c->ev[0], s));
            CU(launch_rowbuild_sigma(c->B, c->d_table, c->n, c->w, c->d, c->K, c->d_anchors, na, c->d_l1, c->d_meta,
                                     c->d_counters, s));
            CU(cudaEventRecord(c->ev[1], s));
            CU(launch_taskscan(c->d_meta, na, c->t, c->d_task_base, s));
            SigmaParams SP{};
            SP.n = c->n;
            SP.m = c->m;
            SP.l = c->l;
            SP.d = c->d;
            SP.w = c->w;
            SP.K = c->K;
            SP.t = c->t;
            SP.sigma = c->sigma;
            SP.prune = c->opt.prune_level;
            SP.table = c->d_table;
            SP.l1_entries = c->d_l1;
            SP.l1_meta = c->d_meta;
            SP.anchor_off = c->d_anchors;
            SP.task_base = c->d_task_base;
            SP.nanchors = na;
            SP.next_task = c->d_task_counter;
            SP.scratch = c->d_scratch;
            SP.scratch_words = c->scratch_words;
            SP.level_cap = c->level_cap;
            SP.node_cap = c->node_cap;
            SP.keys = c->d_keys;
            SP.key_count = c->d_key_count;
            SP.key_cap = c->key_cap;
            SP.counters = c->d_counters;
            SP.error_flag = c->d_err;
            CU(cudaEventRecord(c->ev[2], s));
            if (na > 0) CU(launch_search_sigma(c->B, SP, c->blocks, c->warps, s));
            CU(cudaEventRecord(c->ev[3], s));
        } else {
            CU(launch_encode(c->W, c->d_codes, c->n, c->m, c->l, c->w, c->d_table, c->d_err, s));
            CU(cudaEventRecord(c->ev[0], s));
            CU(launch_rowbuild(c->W, c->d_table, c->n, c->w, c->d, c->K, c->opt.sort_rows, c->d_anchors, na, c->d_l1,
                               c->d_meta, c->d_counters, s));
            CU(cudaEventRecord(c->ev[1], s));
            CU(launch_taskscan(c->d_meta, na, c->t, c->d_task_base, s));
            const uint32_t* task_order = nullptr;
            if (c->d_order && na > 0) {
                uint32_t* k0 = c->d_order;
                const long long oc = c->order_cap;
                CU(launch_taskorder(c->W, c->d_table, c->d_l1, c->d_meta, c->d_anchors, c->d_task_base, na, c->K, oc, k0,
                                    k0 + 2 * oc, s));
                size_t tb = c->order_tmp_bytes;
                CU(cub::DeviceRadixSort::SortPairs(c->d_order_tmp, tb, k0, k0 + oc, k0 + 2 * oc, k0 + 3 * oc,
                                                   static_cast<int>(oc), 0, 8, s));
                task_order = k0 + 3 * oc;
            }
            SearchParams P{};
            P.n = c->n;
            P.m = c->m;
            P.l = c->l;
            P.d = c->d;
            P.w = c->w;
            P.K = c->K;
            P.t = c->t;
            P.prune = c->opt.prune_level;
            P.sort_rows = c->opt.sort_rows;
            P.table = c->d_table;
            P.l1_entries = c->d_l1;
            P.l1_meta = c->d_meta;
            P.anchor_off = c->d_anchors;
            P.task_base = c->d_task_base;
            P.task_order = task_order;
            P.nanchors = na;
            P.task_ai = c->d_task_ai;
            P.task_u = c->d_task_u;
            P.nexplicit = static_cast<long long>(c->task_u.size());
            P.qs = c->d_qs;
            P.qslots = c->d_qslots;
            P.qstate = c->d_qstate;
            P.qcap = c->qcap;
            P.qslot_bytes = c->qslot_bytes;
            P.don_cap = c->don_cap;
            P.qslot_lvl_off = static_cast<int>(task_slot_level_offset(c->W));
            P.donate = std::getenv("PMS8G_NO_DONATE") ? 0 : 1;
            // DFS pushes between starvation checks: 32 for the short pushes of t <= 3 (4: +1.8 % on
            // (17,6)); t >= 4 pushes are long, 4 feeds the tail sooner ((23,9) 29 S1 l-mers 483 -> 444 ms)
            P.don_pushes = c->t >= 4 ? 4 : 32;
            P.don_rounds_mask = 63;
            P.don_burst = 1;
            // generic (two-word / t >= 5) enumeration: a check per round measured slower
            // ((50,21) t=6: 1.89 s vs 1.29 s per 56 S1 l-mers; the node batches get too small)
            P.don_gen_mask = 7;
            if (const char* e = std::getenv("PMS8G_DON_GEN")) P.don_gen_mask = std::max(1, std::atoi(e)) - 1;
            if (const char* e = std::getenv("PMS8G_DON_BURST")) P.don_burst = std::max(1, std::atoi(e));
            if (const char* e = std::getenv("PMS8G_DON_PUSHES")) P.don_pushes = std::max(1, std::atoi(e));
            if (const char* e = std::getenv("PMS8G_LOG_CYCLES")) P.log_cycles = std::atoll(e);
            if (const char* e = std::getenv("PMS8G_DON_ROUNDS")) P.don_rounds_mask = std::max(1, std::atoi(e)) - 1;
            P.lazy = (c->opt.exact_tree || std::getenv("PMS8G_EAGER")) ? 0 : 1;
            P.reorder = (c->opt.exact_tree || std::getenv("PMS8G_NATURAL_ORDER")) ? 0 : 1;
            // the consensus row rule changes the tree (not the motif set): off for exact_tree
            P.cons_rows = (c->opt.prune_level == 2 && !c->opt.exact_tree && !std::getenv("PMS8G_NO_CONS_ROWS")) ? 1 : 0;
                P.plan = c->plan;
            P.scratch = c->d_scratch;
            P.scratch_words = c->scratch_words;
            P.level_cap = c->level_cap;
            P.node_cap = c->node_cap;
            P.keys = c->d_keys;
            P.key_count = c->d_key_count;
            P.key_cap = c->key_cap;
            P.counters = c->d_counters;
            P.error_flag = c->d_err;
            // cross-GPU claims: 4 tasks per NVLink CAS until the last 16 per warp of this device
            P.claim_chunk = 4;
            if (const char* e = std::getenv("PMS8G_CLAIM_CHUNK")) P.claim_chunk = std::max(1, std::atoi(e));
            P.chunk_until = 16ll * c->blocks * c->warps;
            P.jitter_ns = 1000ull * c->opt.jitter_max_us;
            P.jitter_seed = c->opt.jitter_seed;
            P.gqueue = nullptr;
            P.gepoch = 0;
            if (c->opt.queue && attempt == 0) {
                P.gqueue = static_cast<unsigned long long*>(c->opt.queue->dptr);
                P.gepoch = ++c->opt.queue->epoch;
            }
            // a retry (key buffer grown) searches every task locally: the shared
            // counter's epoch stays in step with the other ranks, and this rank's
            // result is a superset of its share (the union is unchanged)
            if (tl_path) {
                P.timeline_cap = 1 << 21;
                CU(cudaMalloc(&d_tl, sizeof(unsigned long long) * 2 * P.timeline_cap));
                P.timeline = d_tl;
            }
            CU(cudaEventRecord(c->ev[2], s));
            // the dynamic shared-memory limit is a per-kernel attribute, shared by
            // every context of this (W, t) build in the process: set it per launch
            if (na > 0) {
                CU(set_search_smem(c->W, c->t, c->smem));
                CU(launch_search(c->W, P, c->blocks, c->warps, c->smem, s));
            }
            CU(cudaEventRecord(c->ev[3], s));
        }
        CU(cudaMemcpyAsync(c->h_counters, c->d_counters, sizeof(unsigned long long) * C_NCTR, cudaMemcpyDeviceToHost,
                           s));
        CU(cudaMemcpyAsync(c->h_counters + C_NCTR, c->d_key_count, sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, s));
        CU(cudaMemcpyAsync(c->h_err, c->d_err, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        CU(cudaGetLastError());
        if (d_tl) {
            const long long ntl = std::min<long long>(static_cast<long long>(c->h_counters[C_TLN]), 1ll << 21);
            std::vector<unsigned long long> h(2 * static_cast<size_t>(ntl));
            CU(cudaMemcpy(h.data(), d_tl, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
            CU(cudaFree(d_tl));
            if (FILE* f = std::fopen(tl_path, "wb")) {
                std::fwrite(h.data(), sizeof(unsigned long long), h.size(), f);
                std::fclose(f);
            }
        }
        if (c->h_err[0] & 1) return fail(err, errlen, PMS8G_ERR_INVALID, "symbol code outside the alphabet");
        // worker failures name the subproblem like run_parallel (src/parallel.cpp:66-86)
        char where[64] = "search";
        if (c->h_err[1] > 0) std::snprintf(where, sizeof where, "subproblem at offset %d", c->h_err[1] - 1);
        if (c->h_err[0] & 2)
            return fail(err, errlen, PMS8G_ERR_RUNTIME, "%s failed: enumeration stack overflow (l=%d, capacity %d nodes)",
                        where, c->l, c->node_cap);
        if (c->h_err[0] & 8)
            return fail(err, errlen, PMS8G_ERR_RUNTIME, "search failed: work queue watchdog fired (no progress)");
        if (c->h_err[0] & 4)
            return fail(err, errlen, PMS8G_ERR_LOGIC, "%s failed: replay of a donated task diverged from its donor",
                        where);
        const long long raw = static_cast<long long>(c->h_counters[C_NCTR]);
        if (c->opt.max_motifs >= 0 && raw > c->opt.max_motifs)
            return fail(err, errlen, PMS8G_ERR_RUNTIME, "motif cap of %lld exceeded",
                        static_cast<long long>(c->opt.max_motifs));
        if (raw > c->key_cap) {
            int rc = ensure_key_capacity(c, raw + raw / 4 + 1024, err, errlen);
            if (rc) return rc;
            continue;  // rerun with room for every raw emission
        }
        // canonical_motif_set: device radix sort + unique
        using K128 = unsigned __int128;
        long long uniq = 0;
        if (raw > 0) {
            size_t bytes = c->cub_bytes;
            CU(cub::DeviceRadixSort::SortKeys(c->d_cub, bytes, reinterpret_cast<K128*>(c->d_keys),
                                              reinterpret_cast<K128*>(c->d_keys_sorted), static_cast<int>(raw), 0,
                                              c->key_bits(), s));
            bytes = c->cub_bytes;
            CU(cub::DeviceSelect::Unique(c->d_cub, bytes, reinterpret_cast<K128*>(c->d_keys_sorted),
                                         reinterpret_cast<K128*>(c->d_keys_unique), c->d_unique_count,
                                         static_cast<int>(raw), s));
            CU(cudaMemcpyAsync(&c->h_counters[C_NCTR + 1], c->d_unique_count, sizeof(long long),
                               cudaMemcpyDeviceToHost, s));
            if (c->opt.reverify) {
                CU(cudaStreamSynchronize(s));
                uniq = static_cast<long long>(c->h_counters[C_NCTR + 1]);
                if (c->sig)
                    CU(launch_reverify_sigma(c->B, c->d_table, c->n, c->w, c->l, c->d, c->d_keys_unique, uniq,
                                             c->d_fail, s));
                else
                    CU(launch_reverify(c->W, c->d_table, c->n, c->w, c->l, c->d, c->d_keys_unique, uniq, c->d_fail,
                                       s));
                CU(cudaMemcpyAsync(c->h_err + 2, c->d_fail, sizeof(int), cudaMemcpyDeviceToHost, s));
            }
            CU(cudaStreamSynchronize(s));
            uniq = static_cast<long long>(c->h_counters[C_NCTR + 1]);
            if (c->opt.reverify && c->h_err[2])
                return fail(err, errlen, PMS8G_ERR_LOGIC, "re-verification failed for a reported motif");
        }
        c->unique_count = uniq;
        // report (RunReport fields, src/parallel.cpp:92-116)
        pms8g_report& R = c->report;
        std::memset(&R, 0, sizeof R);
        R.n = c->n;
        R.m = c->m;
        R.l = c->l;
        R.d = c->d;
        R.sigma = c->sigma;
        R.threshold = c->ref_t;
        R.device_threshold = c->t;
        R.gpus = 1;
        R.subproblems = na;
        R.motif_count = uniq;
        const unsigned long long* h = c->h_counters;
        R.stacks_explored = static_cast<int64_t>(h[C_PUSHES]);
        R.neighborhoods = static_cast<int64_t>(h[C_TUPLES]);
        R.neighbors_visited = static_cast<int64_t>(h[C_LEAVES]);
        R.motifs_emitted = static_cast<int64_t>(h[C_EMITTED]);
        R.filter_slots = static_cast<int64_t>(h[C_SLOTS]);
        R.verify_compares = static_cast<int64_t>(h[C_VCMP]);
        R.enum_nodes = static_cast<int64_t>(h[C_NODES]);
        float ms_rb = 0, ms_search = 0;
        cudaEventElapsedTime(&ms_rb, c->ev[0], c->ev[1]);
        cudaEventElapsedTime(&ms_search, c->ev[2], c->ev[3]);
        const double cf = static_cast<double>(h[C_CLK_FILTER]), cp = static_cast<double>(h[C_CLK_PATTERN]);
        const double frac_pattern = (cf + cp) > 0 ? cp / (cf + cp) : 0.0;
        R.device_seconds = (ms_rb + ms_search) * 1e-3;
        R.pattern_seconds = ms_search * 1e-3 * frac_pattern;
        R.sample_seconds = R.device_seconds - R.pattern_seconds;
        R.device_bytes = c->device_bytes;
        {
            // MemoryBreakdown of the device layout (include/pms8g.h), 8-byte words
            auto words = [](size_t bytes) { return static_cast<uint64_t>((bytes + 7) / 8); };
            const size_t nwarps = static_cast<size_t>(c->blocks) * c->warps;
            const size_t lvl = static_cast<size_t>(std::max(0, c->t - 1)) * c->level_cap * 4 * nwarps;
            R.pair_matrix_words = words(static_cast<size_t>(std::max(1, na)) * c->K * 4);
            R.row_matrix_words = words(lvl);
            R.row_bookkeeping_words =
                words(sizeof(LevelMeta) * std::max(1, na) + sizeof(long long) * (na + 1) +
                      sizeof(uint32_t) * 4 * static_cast<size_t>(c->order_cap) +
                      static_cast<size_t>(c->qcap) * (c->qslot_bytes + sizeof(unsigned int)) +
                      (c->scratch_words * 4 * nwarps - lvl));
            R.packed_words = words(static_cast<size_t>(c->n) * c->m +
                                   static_cast<size_t>(c->K) * (c->sig ? sigma_lmer_bytes(c->B) : lmer_bytes(c->W)));
            R.lookup_table_words = 0;
        }
        R.wall_seconds = now_s() - t0;
        return PMS8G_OK;
    }
    return fail(err, errlen, PMS8G_ERR_RUNTIME, "motif buffer did not converge");
}

}  // namespace
