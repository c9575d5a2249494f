// Host runtime shared by the C-ABI translation units (prover.cpp, comm.cpp,
// ext.cpp): error guard, device buffers, field handle, lanes (stream +
// workspace + pinned staging), the context, and the communicator interface.
#pragma once

#include <sched.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>
#include <nccl.h>

#include <atomic>
#include <condition_variable>

#include <algorithm>
#include <array>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>
#include <set>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges cost nothing unless a profiler injects a tool

#include "dgkr_b200.h"
#include "fe.hpp"
#include "host_core.hpp"
#include "kernels.hpp"

using namespace dgkr_b200;

namespace dgkr_b200 {

/// last error message of a C-ABI call on this thread (dgkr_last_error)
inline thread_local std::string g_err;

/// NVTX range for nsys / ncu --nvtx timelines: gkr_prove, evaluate, the
/// output absorb, each layer and each sum-check phase are named ranges
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

template <class Fn>
int guard(Fn&& fn) {
    try {
        fn();
        return DGKR_OK;
    } catch (const Error& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::bad_alloc& e) {
        g_err = std::string("host allocation failed: ") + e.what();
        return DGKR_CUDA_ERROR;
    } catch (const std::exception& e) {
        g_err = e.what();
        return DGKR_LOGIC_ERROR;
    }
}

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) fail(DGKR_CUDA_ERROR, std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)

inline double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

template <class T>
struct DBuf {
    T* p = nullptr;
    std::size_t n = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    void ensure(std::size_t count) {
        if (count <= n && p) return;
        release();
        CK(cudaMalloc(reinterpret_cast<void**>(&p), std::max<std::size_t>(count, 1) * sizeof(T)));
        n = std::max<std::size_t>(count, 1);
    }
};

inline Fe to_fe(const U256& x) {
    Fe f;
    std::memcpy(f.v, x.w, 32);
    return f;
}
inline U256 to_u256(const Fe& f) {
    U256 x;
    std::memcpy(x.w, f.v, 32);
    return x;
}

inline std::uint32_t log2_exact(std::uint64_t n) {  // circuit.hpp:57-61
    std::uint32_t l = 0;
    while ((std::uint64_t{1} << l) < n) ++l;
    return l;
}
inline std::uint64_t next_pow2(std::uint64_t n) {  // circuit.hpp:43-47
    std::uint64_t p = 1;
    while (p < n) p <<= 1;
    return p;
}

inline void put32(std::vector<std::uint8_t>& out, std::uint32_t v) {
    for (int i = 0; i < 4; ++i) out.push_back(static_cast<std::uint8_t>(v >> (8 * i)));
}

inline void emit(const std::vector<std::uint8_t>& bytes, std::uint8_t* out, std::size_t cap, std::size_t* len) {
    *len = bytes.size();
    if (bytes.size() > cap) fail(DGKR_CAPACITY, "output buffer too small");
    if (!bytes.empty()) std::memcpy(out, bytes.data(), bytes.size());
}

}  // namespace dgkr_b200

// ===========================================================================
// Opaque handles
// ===========================================================================
struct dgkr_field {
    HostField f;
    FieldKind kind = FieldKind::Runtime;
    RtFieldHost rt{};
    U256 fold_pow[8];  // canonical 2^(32k+64) mod p, for the fold constants
    // NTT data (Montgomery): two-adicity s, w of order 2^s, coset shift g =
    // smallest quadratic non-residue (not in any 2-power subgroup), g^-1
    unsigned two_adicity = 0;
    U256 root{}, coset{}, coset_inv{};

    /// w_N for N = 2^log_n (log_n <= two_adicity)
    U256 root_of_unity(unsigned log_n) const {
        if (log_n > two_adicity) fail(DGKR_UNSUPPORTED, "domain larger than the field's 2-adic subgroup");
        U256 w = root;
        for (unsigned i = log_n; i < two_adicity; ++i) w = f.mul(w, w);
        return w;
    }

    /// {c_0..c_7, r} with c_k = mont(r, 2^(32k+64)) (field.cuh FoldConst)
    void fold_const(const U256& r, U256 out[9]) const {
        for (int k = 0; k < 8; ++k) out[k] = f.mul(r, fold_pow[k]);
        out[8] = r;
    }
};

/// Runtime-modulus constants live in one __constant__ block per device,
/// shared by every context and lane of the process on that device, so the
/// upload-skip cache is per device too (device_rt_state): a context that
/// switches moduli re-uploads no matter which context loaded the block last.
/// Concurrent proofs over DIFFERENT runtime moduli on one device are not
/// supported (they would share the constant block); BN254 has immediates.
struct RtState {
    std::mutex mu;
    bool valid = false;
    RtFieldHost cur{};
};

inline RtState* device_rt_state(int device) {
    static RtState states[64];
    if (device < 0 || device >= 64) fail(DGKR_UNSUPPORTED, "device index out of range");
    return &states[device];
}

/// device buffers of one polynomial commitment (pcs.hpp), kept across calls
struct PcsDevice {
    DBuf<Fe> m;                // rows x cols Montgomery
    DBuf<std::uint8_t> nodes;  // 2*cols digests
    DBuf<std::uint8_t> stage;
    DBuf<Fe> comb, beta, eqt;  // open: combined row, beta weights, split-eq tables
    DBuf<EqJob> jobs;
    DBuf<std::uint64_t> path_idx;  // open: node indexes of every spot check's Merkle path
    DBuf<std::uint8_t> path_out;
};

/// device buffers of the NTT / RS / FRI entry points, kept across calls
/// (multi-GiB at C5 sizes: cudaMalloc/cudaFree per call would dominate)
struct NttWs {
    DBuf<std::uint8_t> stage, dbuf;
    DBuf<Fe> x, a, tw, cpow, scratch, twinv;
    std::vector<std::unique_ptr<DBuf<Fe>>> layer;
    std::vector<std::unique_ptr<DBuf<std::uint8_t>>> tree;
    DBuf<std::uint64_t> didx;
    // beacon tree (config C3)
    DBuf<std::uint8_t> b_recs, b_nodes, b_leaves, b_sib, b_zc, b_ok, b_root;
    // polynomial commitment (pcs_commit / pcs_open; a DistPc cluster on this lane)
    PcsDevice pcs;
    // DistPc worker row resident on this lane's device (Montgomery), the
    // source of the peer copy into its cluster leader's matrix
    DBuf<Fe> worker_row;
    DBuf<std::uint8_t> worker_stage;
};

/// Combining scheduler for the serial output absorbs of concurrent proofs
/// (gkr.hpp:189-190: state <- SHA256(state || out_i) for every padded
/// output). One chain is bound by SHA-NI round latency; K chains interleaved
/// in one thread (absorb_chain32_multi) run ~1.5x (one core) to ~2.3x (all
/// cores busy) the absorbs per core (tools/absorb, profiles/r2/absorb_probe.txt).
/// A lane that reaches its absorb queues its job. If a running processor has
/// a free slot, the lane sleeps: that processor takes the job at its next
/// chunk boundary (2^15 absorbs, a few ms) and advances it interleaved with
/// its own. Otherwise the lane becomes a processor itself. A processor whose
/// own job is done hands the others back (state and position travel with the
/// job) and returns; one of their lanes takes over. Every chain's bytes are
/// exactly absorb_chain32's. max_k = 1 disables the interleaving.
struct AbsorbPool {
    struct Job {
        std::uint8_t* state;
        const std::uint8_t* data;
        std::size_t n;
        std::size_t pos = 0;
        bool owned = false;
        bool done = false;
    };
    static constexpr std::size_t kChunk = std::size_t{1} << 15;
    static constexpr int kMaxK = 4;
    int max_k = 1;     // chains per processor (tuning "absorb_chains"; 1 measured best in the C2 stream)
    std::mutex mu;
    std::condition_variable cv;
    std::vector<Job*> pending;  // unowned and unfinished, FIFO
    int spare = 0;              // free slots of the running processors

    void run(std::uint8_t* state, const std::uint8_t* data, std::size_t n) {
        Job me{state, data, n};
        if (n == 0) return;
        std::unique_lock<std::mutex> lk(mu);
        pending.push_back(&me);
        for (;;) {
            if (me.done) return;
            if (!me.owned && spare == 0) {
                std::vector<Job*> mine;
                take(&me, mine);
                fill(mine);
                spare += max_k - static_cast<int>(mine.size());
                lk.unlock();
                process(mine, &me);
                lk.lock();
                continue;
            }
            cv.wait(lk);
        }
    }

private:
    void take(Job* j, std::vector<Job*>& mine) {  // mu held
        pending.erase(std::find(pending.begin(), pending.end(), j));
        j->owned = true;
        mine.push_back(j);
    }
    void fill(std::vector<Job*>& mine) {  // mu held
        while (static_cast<int>(mine.size()) < max_k && !pending.empty()) take(pending.front(), mine);
    }
    void process(std::vector<Job*> mine, Job* me) {
        std::uint8_t* st[kMaxK];
        const std::uint8_t* in[kMaxK];
        for (;;) {
            std::size_t m = kChunk;
            for (Job* j : mine) m = std::min(m, j->n - j->pos);
            for (std::size_t k = 0; k < mine.size(); ++k) {
                st[k] = mine[k]->state;
                in[k] = mine[k]->data + 32 * mine[k]->pos;
            }
            absorb_chain32_multi(st, in, mine.size(), m);
            std::lock_guard<std::mutex> lk(mu);
            spare -= max_k - static_cast<int>(mine.size());  // this processor's slots, re-added below
            bool any_done = false;
            for (Job* j : mine) {
                j->pos += m;
                if (j->pos == j->n) j->done = any_done = true;
            }
            mine.erase(std::remove_if(mine.begin(), mine.end(), [](Job* j) { return j->done; }), mine.end());
            if (me->done) {
                for (Job* j : mine) {  // hand back, progress kept
                    j->owned = false;
                    pending.insert(pending.begin(), j);
                }
                cv.notify_all();
                return;
            }
            fill(mine);
            spare += max_k - static_cast<int>(mine.size());
            if (any_done) cv.notify_all();
        }
    }
};

/// One in-flight proof: a CUDA stream, its reduction workspace, pinned
/// staging and profile counters. A context owns one lane per concurrent
/// proof (lane 0 serves the single-call API).
struct Lane {
    int device = 0;
    int sms = 0;
    int index = 0;
    RtState* rt = nullptr;
    cudaStream_t st = nullptr;
    ReduceWs ws;
    DBuf<Fe> partials, result;
    DBuf<unsigned> counter;
    DBuf<Fe> d_small;      // challenges, points, seeds, finals
    DBuf<int> d_err;
    DBuf<int> d_flag;       // kernel-raised predicate flags (distinct checks)
    Fe* h_small = nullptr;  // pinned mirror of d_small
    TailMailbox* tail_mb = nullptr;      // pinned, mapped: the tail kernel's mailbox (host view)
    TailMailbox* tail_mb_dev = nullptr;  // its device address
    std::uint32_t tail_gen = 0;          // generation of the last tail launch (mailbox tags)
    // pinned staging layout (Fe units): [0] challenge, [1..4) reduction
    // results, [16, 8192) eq-table points/seeds, [8192, 12288) slot values,
    // [12288, 16384) round finals.
    static constexpr std::size_t kSmall = 1 << 14;
    static constexpr std::size_t kEqOff = 16, kEqOff2 = 4112, kVxOff = 8192, kFinalsOff = 12288;
    static constexpr std::size_t kGatherOff = 14336;  // [14336, 16384): all-gathered round sums (<= 682 ranks)
    bool profile_on = false;
    dgkr_profile prof{};
    /// profile-only CUDA-event bracket around a kernel group: tbeg(); ...; tend(prof.x_ms)
    void tbeg() {
        if (profile_on) CK(cudaEventRecord(ev0, st));
    }
    void tend(double& acc) {
        if (!profile_on) return;
        CK(cudaEventRecord(ev1, st));
        CK(cudaEventSynchronize(ev1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, ev0, ev1));
        acc += ms;
    }
    std::unique_ptr<NttWs> ntt_ws;
    NttWs& nttws() {
        if (!ntt_ws) ntt_ws = std::make_unique<NttWs>();
        return *ntt_ws;
    }
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;

    Lane(int dev, int sm_count, int idx, RtState* rts) : device(dev), sms(sm_count), index(idx), rt(rts) {
        CK(cudaSetDevice(device));
        CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        ws.num_sms = sms;
        ws.max_blocks = sms * 8;
        partials.ensure(static_cast<std::size_t>(ws.max_blocks) * 3);
        result.ensure(4);
        counter.ensure(1);
        CK(cudaMemset(counter.p, 0, sizeof(unsigned)));
        ws.partials = partials.p;
        ws.result = result.p;
        ws.counter = counter.p;
        d_small.ensure(kSmall);
        d_err.ensure(1);
        CK(cudaMemset(d_err.p, 0, sizeof(int)));
        d_flag.ensure(2);
        CK(cudaMallocHost(reinterpret_cast<void**>(&h_small), kSmall * sizeof(Fe)));
        CK(cudaHostAlloc(reinterpret_cast<void**>(&tail_mb), sizeof(TailMailbox), cudaHostAllocMapped | cudaHostAllocPortable));
        std::memset(static_cast<void*>(tail_mb), 0, sizeof(TailMailbox));
        CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&tail_mb_dev), tail_mb, 0));
        CK(cudaEventCreate(&ev0));
        CK(cudaEventCreate(&ev1));
        CK(cudaEventCreateWithFlags(&ev_sync, cudaEventBlockingSync | cudaEventDisableTiming));
        if (const char* e = std::getenv("DGKR_SPIN_US")) spin_ms = std::atof(e) * 1e-3;
    }
    Lane(const Lane&) = delete;
    Lane& operator=(const Lane&) = delete;

    ~Lane() {
        for (auto& e : up_ev)
            if (e) cudaEventDestroy(e);
        if (up_ring) cudaFreeHost(up_ring);
        if (ev_sync) cudaEventDestroy(ev_sync);
        if (h_small) cudaFreeHost(h_small);
        if (tail_mb) cudaFreeHost(tail_mb);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        if (st) cudaStreamDestroy(st);
    }

    FieldKind use(const dgkr_field* f) {
        if (f->kind != FieldKind::Bn254) {
            std::lock_guard<std::mutex> lk(rt->mu);
            if (!rt->valid || std::memcmp(&rt->cur, &f->rt, sizeof(RtFieldHost)) != 0) {
                upload_rt_field(f->rt, st);
                CK(cudaStreamSynchronize(st));
                rt->cur = f->rt;
                rt->valid = true;
            }
        }
        return f->kind;
    }

    /// Wait for the stream: poll briefly (round kernels on small tables finish
    /// in microseconds), then block on an event so that waiting lanes leave
    /// the host cores to the lanes running their serial SHA-256 chains.
    void sync() {
        CK(cudaEventRecord(ev_sync, st));
        const double t0 = now_ms();
        for (;;) {
            const cudaError_t q = cudaEventQuery(ev_sync);
            if (q == cudaSuccess) return;
            if (q != cudaErrorNotReady) CK(q);
            if (now_ms() - t0 > spin_ms) break;
            if (tuning().spin_yield) sched_yield();  // leave the core to a lane running its transcript
        }
        CK(cudaEventSynchronize(ev_sync));
    }
    cudaEvent_t ev_sync = nullptr;
    double spin_ms = 1e12;  // measured: polling beats blocking even with 16 lanes (DGKR_SPIN_US to change)

    void begin_call() {
        std::memset(&prof, 0, sizeof(prof));
        prof.total_ms = now_ms();
    }
    void end_call() { prof.total_ms = now_ms() - prof.total_ms; }

    void h2d(void* dst, const void* src, std::size_t n) {
        CK(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, st));
        prof.h2d_bytes += n;
    }
    /// Large pageable uploads: the driver stages pageable memory through its
    /// own pinned buffer at ~11 GB/s on this host (pinned DMA: ~55 GB/s). Here
    /// kUpThreads host threads copy contiguous parts into their own pinned
    /// two-slot rings and enqueue each chunk's DMA on the lane stream, so the
    /// host copies run in parallel and overlap the DMA. Stream order covers
    /// later kernels; a slot is rewritten only after its previous DMA's event.
    /// Pinned sources and small copies take the plain path.
    static constexpr int kUpThreads = 8;
    static constexpr std::size_t kUpChunk = std::size_t{8} << 20;
    std::uint8_t* up_ring = nullptr;  // kUpThreads * 2 * kUpChunk, pinned, lazily
    cudaEvent_t up_ev[kUpThreads * 2] = {};
    bool up_recorded[kUpThreads * 2] = {};
    void h2d_large(void* dst, const void* src, std::size_t n) {
        cudaPointerAttributes at{};
        const bool pinned = cudaPointerGetAttributes(&at, src) == cudaSuccess && at.type == cudaMemoryTypeHost;
        if (!pinned) (void)cudaGetLastError();  // clear a not-registered report
        if (pinned || n < 4 * kUpChunk) {
            h2d(dst, src, n);
            return;
        }
        if (!up_ring) {
            CK(cudaMallocHost(reinterpret_cast<void**>(&up_ring), kUpThreads * 2 * kUpChunk));
            for (auto& e : up_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        const std::size_t part = (n + kUpThreads - 1) / kUpThreads;
        std::vector<std::thread> th;
        std::vector<int> errs(kUpThreads, 0);
        auto work = [&](int k) {
            if (cudaSetDevice(device) != cudaSuccess) {
                errs[k] = 1;
                return;
            }
            const std::size_t b = std::min(n, k * part), e = std::min(n, b + part);
            int slot = 0;
            for (std::size_t off = b; off < e; off += kUpChunk, slot ^= 1) {
                const std::size_t len = std::min(kUpChunk, e - off);
                const int s = 2 * k + slot;
                std::uint8_t* buf = up_ring + static_cast<std::size_t>(s) * kUpChunk;
                if (up_recorded[s] && cudaEventSynchronize(up_ev[s]) != cudaSuccess) {
                    errs[k] = 1;
                    return;
                }
                std::memcpy(buf, static_cast<const std::uint8_t*>(src) + off, len);
                if (cudaMemcpyAsync(static_cast<std::uint8_t*>(dst) + off, buf, len, cudaMemcpyHostToDevice, st) !=
                        cudaSuccess ||
                    cudaEventRecord(up_ev[s], st) != cudaSuccess) {
                    errs[k] = 1;
                    return;
                }
                up_recorded[s] = true;
            }
        };
        for (int k = 1; k < kUpThreads; ++k) th.emplace_back(work, k);
        work(0);
        for (auto& t : th) t.join();
        for (int k = 0; k < kUpThreads; ++k)
            if (errs[k]) fail(DGKR_CUDA_ERROR, std::string("chunked upload: ") + cudaGetErrorString(cudaGetLastError()));
        prof.h2d_bytes += n;
    }
    /// Large downloads into pageable memory, the mirror of h2d_large: chunk
    /// DMAs into per-thread pinned slots on the lane stream, host threads copy
    /// each slot out once its event fires. Returns with the data in dst (the
    /// lane stream has reached the last chunk). Pinned destinations and small
    /// copies take the plain path plus a stream sync.
    void d2h_large(void* dst, const void* src, std::size_t n) {
        cudaPointerAttributes at{};
        const bool pinned = cudaPointerGetAttributes(&at, dst) == cudaSuccess && at.type == cudaMemoryTypeHost;
        if (!pinned) (void)cudaGetLastError();
        if (pinned || n < 4 * kUpChunk) {
            d2h(dst, src, n);
            sync();
            return;
        }
        if (!up_ring) {
            CK(cudaMallocHost(reinterpret_cast<void**>(&up_ring), kUpThreads * 2 * kUpChunk));
            for (auto& e : up_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        const std::size_t part = (n + kUpThreads - 1) / kUpThreads;
        std::vector<std::thread> th;
        std::vector<int> errs(kUpThreads, 0);
        auto work = [&](int k) {
            if (cudaSetDevice(device) != cudaSuccess) {
                errs[k] = 1;
                return;
            }
            const std::size_t b = std::min(n, k * part), e = std::min(n, b + part);
            auto enqueue = [&](std::size_t off, int slot) {
                const int s = 2 * k + slot;
                const std::size_t len = std::min(kUpChunk, e - off);
                if (up_recorded[s] && cudaEventSynchronize(up_ev[s]) != cudaSuccess) return false;
                if (cudaMemcpyAsync(up_ring + static_cast<std::size_t>(s) * kUpChunk,
                                    static_cast<const std::uint8_t*>(src) + off, len, cudaMemcpyDeviceToHost,
                                    st) != cudaSuccess ||
                    cudaEventRecord(up_ev[s], st) != cudaSuccess)
                    return false;
                up_recorded[s] = true;
                return true;
            };
            // two chunks in flight per thread: copy one out while the next lands
            if (b < e && !enqueue(b, 0)) errs[k] = 1;
            if (b + kUpChunk < e && !enqueue(b + kUpChunk, 1)) errs[k] = 1;
            int slot = 0;
            for (std::size_t off = b; off < e && !errs[k]; off += kUpChunk, slot ^= 1) {
                const int s = 2 * k + slot;
                const std::size_t len = std::min(kUpChunk, e - off);
                if (cudaEventSynchronize(up_ev[s]) != cudaSuccess) {
                    errs[k] = 1;
                    break;
                }
                std::memcpy(static_cast<std::uint8_t*>(dst) + off, up_ring + static_cast<std::size_t>(s) * kUpChunk,
                            len);
                if (off + 2 * kUpChunk < e && !enqueue(off + 2 * kUpChunk, slot)) errs[k] = 1;
            }
        };
        for (int k = 1; k < kUpThreads; ++k) th.emplace_back(work, k);
        work(0);
        for (auto& t : th) t.join();
        for (int k = 0; k < kUpThreads; ++k)
            if (errs[k]) fail(DGKR_CUDA_ERROR, std::string("chunked download: ") + cudaGetErrorString(cudaGetLastError()));
        prof.d2h_bytes += n;
    }
    void d2h(void* dst, const void* src, std::size_t n) {
        CK(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, st));
        prof.d2h_bytes += n;
    }
    void launched(std::uint64_t n = 1) { prof.launches += n; }

    void check_err_flag(const char* what) {
        int h = 0;
        CK(cudaMemcpyAsync(&h, d_err.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        sync();
        if (h) {
            CK(cudaMemsetAsync(d_err.p, 0, sizeof(int), st));
            fail(DGKR_INVALID_ARGUMENT, std::string("non-canonical field element encoding (") + what + ")");
        }
    }

    /// canonical bytes (host) -> Montgomery Fe (device)
    void upload_elems(const dgkr_field* f, const std::uint8_t* host, std::uint64_t n, Fe* dst, DBuf<std::uint8_t>& stage) {
        if (n == 0) return;
        const std::size_t bytes = n * f->f.width();
        stage.ensure(bytes);
        h2d_large(stage.p, host, bytes);
        launch_from_canonical(use(f), stage.p, static_cast<int>(f->f.width()), dst, n, d_err.p, st);
        launched();
        check_err_flag("input tables");
    }
};

/// The context is lane 0 itself; extra lanes (concurrent proofs) are
/// created on demand and share the runtime-field state.
struct dgkr_ctx : Lane {
    AbsorbPool absorb_pool;  // output absorbs of the concurrent proofs of a stream
    std::mutex lanes_mu;
    std::vector<std::unique_ptr<Lane>> extra;  // lanes 1..
    cudaEvent_t user_ev[8] = {};

    dgkr_ctx(int dev, int sm_count) : Lane(dev, sm_count, 0, device_rt_state(dev)) {}

    Lane* lane(int i) {
        if (i == 0) return this;
        std::lock_guard<std::mutex> lk(lanes_mu);
        while (static_cast<int>(extra.size()) < i)
            extra.push_back(std::make_unique<Lane>(device, sms, static_cast<int>(extra.size()) + 1, rt));
        return extra[i - 1].get();
    }

    ~dgkr_ctx() {
        for (auto& e : user_ev)
            if (e) cudaEventDestroy(e);
    }
};

/// largest communicator: the per-round all-gather of up to 3 round sums per
/// rank lands in h_small[kGatherOff, kSmall)
constexpr int kMaxCommWorld = static_cast<int>((Lane::kSmall - Lane::kGatherOff) / 3);

// ===========================================================================
// Device communication for the data-parallel (multi-GPU) prover. The protocol
// code is shared; only the transport differs (comm.hpp):
//   NcclComm    one process per GPU, NCCL over NVLink/NVSwitch
//   ShmComm     one process per GPU on one node, POSIX shared memory per lane
//   ThreadComm  ranks as host threads driving lanes of ONE GPU, exchanging
//               through host memory at barriers (tests the distributed
//               protocol on a single device; no kernel ever waits on another)
// Per sum-check round the only traffic is an all-gather of 2-3 field elements
// per rank (cluster.hpp:272-286); at each phase boundary an all-gather of the
// final table values (cluster.hpp:295-309).
// ===========================================================================
struct dgkr_comm {
    int rank = 0;
    int world = 1;
    DBuf<std::uint8_t> scratch;
    virtual ~dgkr_comm() = default;
    /// d_recv (device) = concatenation over ranks of each rank's d_send
    virtual void allgather(const void* d_send, void* d_recv, std::size_t bytes, Lane* L) = 0;
    /// h_recv (host) = concatenation over ranks of each rank's d_send
    virtual void allgather_to_host(const void* d_send, void* h_recv, std::size_t bytes, Lane* L) {
        scratch.ensure(static_cast<std::size_t>(world) * bytes);
        allgather(d_send, scratch.p, bytes, L);
        L->d2h(h_recv, scratch.p, static_cast<std::size_t>(world) * bytes);
        L->sync();
    }
    /// rank `root`: h_recv (host) = concatenation over ranks of d_send; others: untouched
    virtual void gather_to_root_host(const void* d_send, void* h_recv, std::size_t bytes, Lane* L, int root) = 0;
    /// every rank's h (host, `bytes`) = rank `root`'s h
    virtual void broadcast_host(void* h, std::size_t bytes, Lane* L, int root) = 0;
};
