// pms8g_multi.cu — run_parallel over several GPUs from one blocking C call.
//
// The reference's run_parallel (src/parallel.cpp:35-118) is one blocking call
// that owns its worker team: the workers pull S1 offsets from a shared atomic
// job counter (:54-60), every worker's motifs are merged in job order and
// canonicalised (:88-90). Here the workers are GPUs, driven by one host
// thread each:
//   * one device context per GPU (pms8g_ctx: encode, row build, persistent
//     search, device sort/unique), all searching every S1 l-mer but claiming
//     (S1 l-mer, depth-1 branch) tasks from ONE epoch-tagged counter in the
//     first device's HBM, reached by the others over NVLink/NVSwitch peer
//     access (the same counter protocol as pms8g_queue_*); if
//     some device cannot reach it, the S1 offsets are split statically
//     (offset % N == rank) instead;
//   * the union of the per-GPU motif sets: ncclAllGather of the padded key
//     buffers over NVLink when the devices are distinct and NCCL is loadable
//     (dlopen: no link-time dependency, and a process that already loaded
//     torch's NCCL reuses it), else peer copies into the first device; then
//     one device sort + unique (grow-only scratch, allocated once).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "pms8g_internal.h"

using namespace pms8g;

#define CU(call) PMS8G_CU(call)

namespace {

// ---- NCCL through dlopen (types as in nccl.h; only the calls used here)
typedef struct ncclComm* ncclComm_t;
typedef int ncclResult_t;  // ncclSuccess == 0
enum { kNcclUint8 = 1 };   // ncclDataType_t: ncclInt8 = 0, ncclUint8 = 1
struct Nccl {
    bool ok = false;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        if (std::getenv("PMS8G_NO_NCCL")) return;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);  // already loaded (torch)?
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        n.CommInitAll = reinterpret_cast<decltype(n.CommInitAll)>(dlsym(h, "ncclCommInitAll"));
        n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
        n.AllGather = reinterpret_cast<decltype(n.AllGather)>(dlsym(h, "ncclAllGather"));
        n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(dlsym(h, "ncclGroupStart"));
        n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
        n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
        n.ok = n.CommInitAll && n.CommDestroy && n.AllGather && n.GroupStart && n.GroupEnd && n.GetErrorString;
    });
    return n;
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

struct pms8g_multi {
    int n = 0, m = 0, l = 0, d = 0;
    std::string alphabet;
    std::vector<int> devices;
    std::vector<pms8g_ctx*> ctx;
    std::vector<pms8g_queue*> queues;  // one view of the shared counter per context
    void* counter = nullptr;           // on devices[0]
    bool shared_queue = false;         // else static split
    bool use_nccl = false;
    std::vector<ncclComm_t> comms;
    std::vector<cudaStream_t> xstreams;  // exchange streams (one per device)
    std::vector<void*> send, recv;       // NCCL buffers per device (grow-only)
    long long xcap = 0;                  // keys per rank the buffers hold
    void* gathered = nullptr;            // keys of every device, on devices[0]
    void* merged = nullptr;
    long long gcap = 0;
    MergeScratch scratch;
    std::string exchange;  // "nccl-allgather" | "peer-copy"
};

namespace {

void destroy_multi(pms8g_multi* h) {
    if (!h) return;
    for (pms8g_ctx* c : h->ctx) pms8g_ctx_destroy(c);
    for (pms8g_queue* q : h->queues) delete q;  // borrowed views (owner 2)
    for (size_t i = 0; i < h->devices.size(); ++i) {
        cudaSetDevice(h->devices[i]);
        if (i < h->send.size() && h->send[i]) cudaFree(h->send[i]);
        if (i < h->recv.size() && h->recv[i]) cudaFree(h->recv[i]);
        if (i < h->xstreams.size() && h->xstreams[i]) cudaStreamDestroy(h->xstreams[i]);
    }
    if (h->use_nccl)
        for (ncclComm_t c : h->comms) nccl().CommDestroy(c);
    if (!h->devices.empty()) {
        cudaSetDevice(h->devices[0]);
        if (h->counter) cudaFree(h->counter);
        if (h->gathered) cudaFree(h->gathered);
        if (h->merged) cudaFree(h->merged);
    }
    merge_scratch_free(h->scratch);
    delete h;
}

}  // namespace

extern "C" {

int pms8g_multi_create(int n, int m, int l, int d, const char* alphabet, const pms8g_options* opt_in,
                       const int* devices, int ndevices, pms8g_multi** out, char* err, size_t errlen) {
    *out = nullptr;
    if (ndevices < 1 || !devices) return fail(err, errlen, PMS8G_ERR_INVALID, "need at least one device");
    pms8g_options opt;
    if (opt_in) opt = *opt_in;
    else pms8g_default_options(&opt);
    if (opt.queue || opt.shard_count > 1)
        return fail(err, errlen, PMS8G_ERR_INVALID, "multi-GPU runs own their queue: no queue or sharding options");
    if (opt.branches) return fail(err, errlen, PMS8G_ERR_INVALID, "explicit branches are single-device only");
    int ndev = 0;
    cudaError_t ce = cudaGetDeviceCount(&ndev);
    if (ce != cudaSuccess || ndev == 0)
        return fail(err, errlen, PMS8G_ERR_CUDA, "no CUDA device available (%s); the GPU path has no CPU fallback",
                    cudaGetErrorString(ce));
    for (int i = 0; i < ndevices; ++i)
        if (devices[i] < 0 || devices[i] >= ndev)
            return fail(err, errlen, PMS8G_ERR_INVALID, "device %d not present (%d devices)", devices[i], ndev);
    auto* h = new pms8g_multi();
    h->n = n;
    h->m = m;
    h->l = l;
    h->d = d;
    h->alphabet = alphabet ? alphabet : "ACGT";
    h->devices.assign(devices, devices + ndevices);
    const int N = ndevices;
    // the shared claim counter lives in the first device's HBM; every other
    // device must reach it by peer access (or be the same device)
    bool reach = true;
    for (int i = 1; i < N; ++i) {
        if (h->devices[i] == h->devices[0]) continue;
        int can = 0;
        cudaDeviceCanAccessPeer(&can, h->devices[i], h->devices[0]);
        if (!can) reach = false;
    }
    if (std::getenv("PMS8G_MULTI_STATIC")) reach = false;
    // alphabets of 5+ symbols run the B-plane search, which claims from its
    // device-local counter: split the S1 offsets statically
    if (alphabet && std::strlen(alphabet) > 4) reach = false;
    int rc = PMS8G_OK;
    auto bail = [&](int code) {
        destroy_multi(h);
        return code;
    };
    if (reach && N > 1) {
        if (cudaSetDevice(h->devices[0]) != cudaSuccess || cudaMalloc(&h->counter, 256) != cudaSuccess ||
            cudaMemset(h->counter, 0, 256) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess)
            return bail(fail(err, errlen, PMS8G_ERR_CUDA, "cannot allocate the shared claim counter"));
        for (int i = 1; i < N; ++i) {
            if (h->devices[i] == h->devices[0]) continue;
            cudaSetDevice(h->devices[i]);
            const cudaError_t pe = cudaDeviceEnablePeerAccess(h->devices[0], 0);
            if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) {
                cudaGetLastError();
                reach = false;
            }
        }
    }
    h->shared_queue = reach && N > 1;
    for (int i = 0; i < N; ++i) {
        pms8g_options o = opt;
        o.device = h->devices[i];
        if (h->shared_queue) {
            auto* q = new pms8g_queue();
            q->dptr = h->counter;
            q->device = h->devices[i];
            q->owner = 2;
            h->queues.push_back(q);
            o.queue = q;
        } else if (N > 1) {
            o.shard_rank = i;
            o.shard_count = N;
        }
        pms8g_ctx* c = nullptr;
        if ((rc = pms8g_ctx_create(n, m, l, d, alphabet, &o, &c, err, errlen)) != PMS8G_OK) return bail(rc);
        h->ctx.push_back(c);
    }
    // exchange: NCCL over distinct devices, else peer copies
    bool distinct = true;
    for (int i = 0; i < N; ++i)
        for (int j = 0; j < i; ++j)
            if (h->devices[i] == h->devices[j]) distinct = false;
    h->xstreams.assign(N, nullptr);
    for (int i = 0; i < N; ++i) {
        cudaSetDevice(h->devices[i]);
        if (cudaStreamCreateWithFlags(&h->xstreams[i], cudaStreamNonBlocking) != cudaSuccess)
            return bail(fail(err, errlen, PMS8G_ERR_CUDA, "cannot create exchange stream"));
    }
    h->send.assign(N, nullptr);
    h->recv.assign(N, nullptr);
    if (distinct && nccl().ok) {
        h->comms.assign(N, nullptr);
        const ncclResult_t r = nccl().CommInitAll(h->comms.data(), N, h->devices.data());
        if (r == 0) {
            h->use_nccl = true;
        } else {
            h->comms.clear();
        }
    }
    h->exchange = h->use_nccl ? "nccl-allgather" : "peer-copy";
    *out = h;
    return PMS8G_OK;
}

void pms8g_multi_destroy(pms8g_multi* h) { destroy_multi(h); }

const char* pms8g_multi_exchange(const pms8g_multi* h) { return h ? h->exchange.c_str() : ""; }

int pms8g_multi_run(pms8g_multi* h, const uint8_t* codes, pms8g_result* out, char* err, size_t errlen) {
    std::memset(out, 0, sizeof *out);
    const double t0 = now_s();
    const int N = static_cast<int>(h->devices.size());
    // one host thread per device: load the codes, run the whole pipeline
    std::vector<int> rcs(N, PMS8G_OK);
    std::vector<std::string> errs(N, std::string(512, '\0'));
    {
        std::vector<std::thread> th;
        for (int i = 0; i < N; ++i)
            th.emplace_back([&, i] {
                char* e = errs[i].data();
                rcs[i] = pms8g_ctx_load_codes(h->ctx[i], codes, 0, e, 512);
                if (!rcs[i]) rcs[i] = pms8g_ctx_run(h->ctx[i], e, 512);
            });
        for (auto& t : th) t.join();
    }
    for (int i = 0; i < N; ++i)
        if (rcs[i]) return fail(err, errlen, rcs[i], "device %d: %s", h->devices[i], errs[i].c_str());
    // per-device unique keys (device pointers + counts, known on the host)
    std::vector<const uint64_t*> keys(N);
    std::vector<long long> cnt(N);
    long long maxc = 0, total = 0;
    for (int i = 0; i < N; ++i) {
        int64_t c = 0;
        pms8g_ctx_keys(h->ctx[i], &keys[i], &c);
        cnt[i] = c;
        maxc = std::max(maxc, cnt[i]);
        total += cnt[i];
    }
    const int root = h->devices[0];
    CU(cudaSetDevice(root));
    if (total > h->gcap || !h->gathered) {
        if (h->gathered) cudaFree(h->gathered);
        if (h->merged) cudaFree(h->merged);
        h->gathered = h->merged = nullptr;
        h->gcap = std::max<long long>(std::max<long long>(total, 1024), 2 * h->gcap);
        CU(cudaMalloc(&h->gathered, 16 * static_cast<size_t>(h->gcap)));
        CU(cudaMalloc(&h->merged, 16 * static_cast<size_t>(h->gcap)));
    }
    if (h->use_nccl && N > 1 && maxc > 0) {
        // allgather of padded key blocks (maxc keys per rank) over NVLink
        if (maxc > h->xcap) {
            const long long cap = std::max<long long>(maxc, std::max<long long>(1024, 2 * h->xcap));
            for (int i = 0; i < N; ++i) {
                CU(cudaSetDevice(h->devices[i]));
                if (h->send[i]) cudaFree(h->send[i]);
                if (h->recv[i]) cudaFree(h->recv[i]);
                h->send[i] = h->recv[i] = nullptr;
                CU(cudaMalloc(&h->send[i], 16 * static_cast<size_t>(cap)));
                CU(cudaMalloc(&h->recv[i], 16 * static_cast<size_t>(cap) * N));
            }
            h->xcap = cap;
        }
        for (int i = 0; i < N; ++i) {
            CU(cudaSetDevice(h->devices[i]));
            if (cnt[i] > 0)
                CU(cudaMemcpyAsync(h->send[i], keys[i], 16 * static_cast<size_t>(cnt[i]), cudaMemcpyDeviceToDevice,
                                   h->xstreams[i]));
        }
        nccl().GroupStart();
        for (int i = 0; i < N; ++i) {
            cudaSetDevice(h->devices[i]);
            const ncclResult_t r = nccl().AllGather(h->send[i], h->recv[i], 16 * static_cast<size_t>(maxc), kNcclUint8,
                                                    h->comms[i], h->xstreams[i]);
            if (r != 0) {
                nccl().GroupEnd();
                return fail(err, errlen, PMS8G_ERR_RUNTIME, "ncclAllGather failed: %s", nccl().GetErrorString(r));
            }
        }
        const ncclResult_t r = nccl().GroupEnd();
        if (r != 0) return fail(err, errlen, PMS8G_ERR_RUNTIME, "ncclAllGather failed: %s", nccl().GetErrorString(r));
        // compact the valid prefix of every rank's block on the root
        CU(cudaSetDevice(root));
        long long off = 0;
        for (int i = 0; i < N; ++i) {
            if (cnt[i] > 0)
                CU(cudaMemcpyAsync(static_cast<char*>(h->gathered) + 16 * off,
                                   static_cast<char*>(h->recv[0]) + 16 * static_cast<size_t>(maxc) * i,
                                   16 * static_cast<size_t>(cnt[i]), cudaMemcpyDeviceToDevice, h->xstreams[0]));
            off += cnt[i];
        }
    } else {
        long long off = 0;
        for (int i = 0; i < N; ++i) {
            if (cnt[i] > 0)
                CU(cudaMemcpyPeerAsync(static_cast<char*>(h->gathered) + 16 * off, root, keys[i], h->devices[i],
                                       16 * static_cast<size_t>(cnt[i]), h->xstreams[0]));
            off += cnt[i];
        }
    }
    long long uniq = 0;
    int rc = merge_keys_with(h->scratch, h->gathered, total, h->merged, &uniq, h->xstreams[0], err, errlen);
    if (rc) return rc;
    std::vector<uint64_t> hk(2 * static_cast<size_t>(std::max(0ll, uniq)));
    if (uniq > 0) {
        CU(cudaMemcpyAsync(hk.data(), h->merged, 16 * static_cast<size_t>(uniq), cudaMemcpyDeviceToHost,
                           h->xstreams[0]));
        CU(cudaStreamSynchronize(h->xstreams[0]));
    }
    out->l = h->l;
    out->count = uniq;
    out->motifs = static_cast<char*>(std::malloc(static_cast<size_t>(uniq) * h->l + 1));
    if (!out->motifs) return fail(err, errlen, PMS8G_ERR_RUNTIME, "cannot allocate motif buffer");
    pms8g_decode_keys(hk.data(), uniq, h->l, h->alphabet.c_str(), out->motifs);
    out->motifs[static_cast<size_t>(uniq) * h->l] = 0;
    // report: the run as a whole (counters summed over devices, RunReport
    // semantics of src/parallel.cpp:92-116)
    pms8g_report R{};
    for (int i = 0; i < N; ++i) {
        const pms8g_report* r = nullptr;
        pms8g_ctx_report(h->ctx[i], &r);
        if (i == 0) {
            R = *r;
            continue;
        }
        R.stacks_explored += r->stacks_explored;
        R.neighborhoods += r->neighborhoods;
        R.neighbors_visited += r->neighbors_visited;
        R.motifs_emitted += r->motifs_emitted;
        R.filter_slots += r->filter_slots;
        R.verify_compares += r->verify_compares;
        R.enum_nodes += r->enum_nodes;
        R.device_bytes += r->device_bytes;
        R.pair_matrix_words += r->pair_matrix_words;
        R.row_matrix_words += r->row_matrix_words;
        R.row_bookkeeping_words += r->row_bookkeeping_words;
        R.packed_words += r->packed_words;
        R.device_seconds = std::max(R.device_seconds, r->device_seconds);
        R.sample_seconds = std::max(R.sample_seconds, r->sample_seconds);
        R.pattern_seconds = std::max(R.pattern_seconds, r->pattern_seconds);
        if (!h->shared_queue) R.subproblems += r->subproblems;
    }
    R.gpus = N;
    R.motif_count = uniq;
    R.wall_seconds = now_s() - t0;
    out->report = R;
    return PMS8G_OK;
}

int pms8g_solve_multi(const uint8_t* codes, int n, int m, int l, int d, const char* alphabet,
                      const pms8g_options* opt_in, const int* devices, int ndevices, pms8g_result* out, char* err,
                      size_t errlen) {
    // one cached handle per process (like pms8g_solve's context cache): the
    // device contexts, NCCL communicators and exchange buffers persist across
    // calls of the same shape and device list
    static std::mutex mu;
    static pms8g_multi* cache = nullptr;
    static std::vector<int> cache_devs;
    static pms8g_options cache_opt{};
    std::memset(out, 0, sizeof *out);
    pms8g_options opt;
    if (opt_in) opt = *opt_in;
    else pms8g_default_options(&opt);
    if (n > 32)  // MAXN: search the first 32 sequences on the GPUs, scan the rest (pms8g_capi.cu)
        return solve_many_sequences(codes, n, m, l, d, alphabet, opt, out, err, errlen,
                                    [&](const pms8g_options& o, pms8g_result* r) {
                                        return pms8g_solve_multi(codes, 32, m, l, d, alphabet, &o, devices,
                                                                 ndevices, r, err, errlen);
                                    });
    std::lock_guard<std::mutex> g(mu);
    const std::vector<int> devs(devices, devices + std::max(0, ndevices));
    const bool same = cache && cache->n == n && cache->m == m && cache->l == l && cache->d == d &&
                      cache->alphabet == (alphabet ? alphabet : "ACGT") && cache_devs == devs && !opt.anchors &&
                      std::memcmp(&cache_opt, &opt, sizeof opt) == 0;
    pms8g_multi* h = same ? cache : nullptr;
    if (!h) {
        const int rc = pms8g_multi_create(n, m, l, d, alphabet, &opt, devices, ndevices, &h, err, errlen);
        if (rc) return rc;
        if (!opt.anchors) {
            destroy_multi(cache);
            cache = h;
            cache_devs = devs;
            cache_opt = opt;
        }
    }
    const int rc = pms8g_multi_run(h, codes, out, err, errlen);
    if (h != cache) destroy_multi(h);
    return rc;
}

}  // extern "C"
