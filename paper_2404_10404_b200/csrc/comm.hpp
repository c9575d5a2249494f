// Transports behind dgkr_comm (runtime.hpp): ranks as host threads of one
// process (ThreadComm), one-node processes over POSIX shared memory
// (ShmComm), and NCCL over NVLink (NcclComm, libnccl resolved with dlopen).
#pragma once
#include <dlfcn.h>
#include <fcntl.h>
#include <nccl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <condition_variable>
#include <thread>

#include "runtime.hpp"

namespace dgkr_b200 {

struct ThreadGroup {
    int world = 1;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    std::uint64_t gen = 0;
    std::vector<std::uint8_t> buf;
    bool aborted = false;
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        if (aborted) fail(DGKR_COMM_ERROR, "thread group aborted");
        const std::uint64_t g = gen;
        if (++arrived == world) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g || aborted; });
            if (aborted) fail(DGKR_COMM_ERROR, "thread group aborted");
        }
    }
    void abort() {
        std::lock_guard<std::mutex> lk(mu);
        aborted = true;
        cv.notify_all();
    }
};

struct ThreadComm : dgkr_comm {
    ThreadGroup* g = nullptr;
    void stage(std::size_t bytes) {
        g->barrier();  // everyone is done with the previous contents
        if (rank == 0 && g->buf.size() < static_cast<std::size_t>(world) * bytes) g->buf.resize(world * bytes);
        g->barrier();
    }
    void allgather(const void* d_send, void* d_recv, std::size_t bytes, Lane* L) override {
        stage(bytes);
        L->d2h(g->buf.data() + rank * bytes, d_send, bytes);
        L->sync();
        g->barrier();
        L->h2d(d_recv, g->buf.data(), world * bytes);
        L->sync();
    }
    void allgather_to_host(const void* d_send, void* h_recv, std::size_t bytes, Lane* L) override {
        stage(bytes);
        L->d2h(g->buf.data() + rank * bytes, d_send, bytes);
        L->sync();
        g->barrier();
        std::memcpy(h_recv, g->buf.data(), world * bytes);
    }
    void gather_to_root_host(const void* d_send, void* h_recv, std::size_t bytes, Lane* L, int root) override {
        stage(bytes);
        L->d2h(g->buf.data() + rank * bytes, d_send, bytes);
        L->sync();
        g->barrier();
        if (rank == root) std::memcpy(h_recv, g->buf.data(), world * bytes);
    }
    void broadcast_host(void* h, std::size_t bytes, Lane*, int root) override {
        stage(bytes);
        if (rank == root) std::memcpy(g->buf.data(), h, bytes);
        g->barrier();
        if (rank != root) std::memcpy(h, g->buf.data(), bytes);
    }
};

// One-node multi-process transport: a POSIX shared-memory segment per lane
// (ranks = processes, one per GPU). The per-round payloads are already on the
// host (the transcript needs them there), so a host exchange is the
// lowest-latency path; every lane has its own segment and barrier, so lanes
// never order-depend on one another (no cross-lane deadlock, unlike sharing
// NCCL communicators between concurrently progressing lanes).
struct ShmHeader {
    std::atomic<std::uint64_t> arrived;
    std::atomic<std::uint64_t> gen;
    std::atomic<std::uint32_t> aborted;
    std::uint32_t world;
    std::uint64_t slot_bytes;
};

struct ShmComm : dgkr_comm {
    ShmHeader* hdr = nullptr;
    std::uint8_t* data = nullptr;  // world * slot_bytes
    std::size_t map_bytes = 0;
    std::string name;
    bool owner = false;
    // pinned bounce buffer (slot_bytes): device <-> slot copies go through it
    // as DMA + memcpy instead of the driver's pageable staging
    std::uint8_t* bounce = nullptr;
    ~ShmComm() override {
        if (bounce) cudaFreeHost(bounce);
        if (hdr) munmap(hdr, map_bytes);
        if (owner) shm_unlink(name.c_str());
    }
    void barrier() {
        const std::uint64_t g = hdr->gen.load(std::memory_order_acquire);
        if (hdr->arrived.fetch_add(1, std::memory_order_acq_rel) + 1 == static_cast<std::uint64_t>(world)) {
            hdr->arrived.store(0, std::memory_order_relaxed);
            hdr->gen.fetch_add(1, std::memory_order_acq_rel);
            return;
        }
        for (std::uint64_t spins = 0; hdr->gen.load(std::memory_order_acquire) == g; ++spins) {
            if (hdr->aborted.load(std::memory_order_relaxed)) fail(DGKR_COMM_ERROR, "peer rank aborted");
            if (spins > 2000) std::this_thread::yield();
        }
    }
    std::uint8_t* slot(int r) { return data + static_cast<std::size_t>(r) * hdr->slot_bytes; }
    void need(std::size_t bytes) const {
        if (bytes > hdr->slot_bytes) fail(DGKR_CAPACITY, "shm slot too small for this exchange");
    }
    /// device -> own slot through the pinned bounce buffer (the copy runs
    /// before the barrier that releases the slot)
    void stage_send(const void* d_send, std::size_t bytes, Lane* L) {
        if (!bounce) fail(DGKR_INVALID_ARGUMENT, "shared-memory communicator created without a context");
        L->d2h(bounce, d_send, bytes);  // counted in the lane profile
        L->sync();
        barrier();  // previous contents consumed
        std::memcpy(slot(rank), bounce, bytes);
        barrier();
    }
    void allgather(const void* d_send, void* d_recv, std::size_t bytes, Lane* L) override {
        need(bytes);
        if (bytes * static_cast<std::size_t>(world) > hdr->slot_bytes) fail(DGKR_CAPACITY, "shm slot too small");
        stage_send(d_send, bytes, L);
        for (int r = 0; r < world; ++r) std::memcpy(bounce + r * bytes, slot(r), bytes);
        L->h2d(d_recv, bounce, static_cast<std::size_t>(world) * bytes);
        L->sync();
    }
    /// chunked through the slots when larger than one (the early-boundary table gather)
    void allgather_to_host(const void* d_send, void* h_recv, std::size_t bytes, Lane* L) override {
        const std::size_t chunk = hdr->slot_bytes;
        std::size_t off = 0;
        do {
            const std::size_t nb = std::min(chunk, bytes - off);
            stage_send(static_cast<const std::uint8_t*>(d_send) + off, nb, L);
            for (int r = 0; r < world; ++r)
                std::memcpy(static_cast<std::uint8_t*>(h_recv) + r * bytes + off, slot(r), nb);
            off += nb;
        } while (off < bytes);
    }
    /// chunked through the slots (the claimed outputs exceed a slot): the
    /// segment stays small however large a rank's share of the outputs is
    void gather_to_root_host(const void* d_send, void* h_recv, std::size_t bytes, Lane* L, int root) override {
        const std::size_t chunk = hdr->slot_bytes;
        std::size_t off = 0;
        do {
            const std::size_t nb = std::min(chunk, bytes - off);
            stage_send(static_cast<const std::uint8_t*>(d_send) + off, nb, L);
            if (rank == root)
                for (int r = 0; r < world; ++r)
                    std::memcpy(static_cast<std::uint8_t*>(h_recv) + r * bytes + off, slot(r), nb);
            off += nb;
        } while (off < bytes);
    }
    void broadcast_host(void* h, std::size_t bytes, Lane*, int root) override {
        need(bytes);
        barrier();
        if (rank == root) std::memcpy(slot(root), h, bytes);
        barrier();
        if (rank != root) std::memcpy(h, slot(root), bytes);
    }
    /// host-only exchange (tests the transport without a GPU)
    void allgather_host(const void* in, std::size_t bytes, void* out) {
        need(bytes);
        barrier();
        std::memcpy(slot(rank), in, bytes);
        barrier();
        for (int r = 0; r < world; ++r) std::memcpy(static_cast<std::uint8_t*>(out) + r * bytes, slot(r), bytes);
    }
};

// NCCL is resolved at run time (dlopen) so the library loads without it;
// torch's bundled libnccl.so.2 is picked up when already loaded.
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    const char* (*errStr)(ncclResult_t) = nullptr;
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*bcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    bool load() {
        if (h) return true;
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (h) break;
        }
        if (!h) return false;
        getUniqueId = reinterpret_cast<decltype(getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        commInitRank = reinterpret_cast<decltype(commInitRank)>(dlsym(h, "ncclCommInitRank"));
        allGather = reinterpret_cast<decltype(allGather)>(dlsym(h, "ncclAllGather"));
        commDestroy = reinterpret_cast<decltype(commDestroy)>(dlsym(h, "ncclCommDestroy"));
        errStr = reinterpret_cast<decltype(errStr)>(dlsym(h, "ncclGetErrorString"));
        send = reinterpret_cast<decltype(send)>(dlsym(h, "ncclSend"));
        recv = reinterpret_cast<decltype(recv)>(dlsym(h, "ncclRecv"));
        bcast = reinterpret_cast<decltype(bcast)>(dlsym(h, "ncclBroadcast"));
        groupStart = reinterpret_cast<decltype(groupStart)>(dlsym(h, "ncclGroupStart"));
        groupEnd = reinterpret_cast<decltype(groupEnd)>(dlsym(h, "ncclGroupEnd"));
        return getUniqueId && commInitRank && allGather && commDestroy && errStr && send && recv && bcast &&
               groupStart && groupEnd;
    }
};
inline NcclApi g_nccl;

#define NCK(x)                                                                                         \
    do {                                                                                               \
        ncclResult_t r_ = (x);                                                                         \
        if (r_ != ncclSuccess) fail(DGKR_COMM_ERROR, std::string(#x) + ": " + g_nccl.errStr(r_));     \
    } while (0)

struct NcclComm : dgkr_comm {
    ncclComm_t comm = nullptr;
    ~NcclComm() override {
        if (comm) g_nccl.commDestroy(comm);
    }
    void allgather(const void* d_send, void* d_recv, std::size_t bytes, Lane* L) override {
        NCK(g_nccl.allGather(d_send, d_recv, bytes, ncclUint8, comm, L->st));
    }
    void gather_to_root_host(const void* d_send, void* h_recv, std::size_t bytes, Lane* L, int root) override {
        if (rank == root) scratch.ensure(static_cast<std::size_t>(world) * bytes);
        NCK(g_nccl.groupStart());
        if (rank == root) {
            for (int r = 0; r < world; ++r)
                if (r != root) NCK(g_nccl.recv(scratch.p + r * bytes, bytes, ncclUint8, r, comm, L->st));
        } else {
            NCK(g_nccl.send(d_send, bytes, ncclUint8, root, comm, L->st));
        }
        NCK(g_nccl.groupEnd());
        if (rank == root) {
            CK(cudaMemcpyAsync(scratch.p + static_cast<std::size_t>(root) * bytes, d_send, bytes,
                               cudaMemcpyDeviceToDevice, L->st));
            L->d2h(h_recv, scratch.p, static_cast<std::size_t>(world) * bytes);
        }
        L->sync();
    }
    void broadcast_host(void* h, std::size_t bytes, Lane* L, int root) override {
        bc.ensure(bytes);
        if (rank == root) L->h2d(bc.p, h, bytes);
        NCK(g_nccl.bcast(bc.p, bc.p, bytes, ncclUint8, root, comm, L->st));
        if (rank != root) L->d2h(h, bc.p, bytes);
        L->sync();
    }
    DBuf<std::uint8_t> bc;
};

}  // namespace dgkr_b200
