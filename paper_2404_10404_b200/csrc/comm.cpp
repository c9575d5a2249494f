// C ABI of the communicators (comm.hpp): NCCL ids and communicators, the
// shared-memory transport and its host-only test hook.
#include <cstring>
#include <memory>
#include <string>

#include "comm.hpp"
#include "dgkr_b200.h"

int dgkr_comm_nccl_unique_id(std::uint8_t* out128) {
    return guard([&] {
        if (!g_nccl.load()) fail(DGKR_COMM_ERROR, "libnccl.so.2 not found");
        ncclUniqueId id;
        NCK(g_nccl.getUniqueId(&id));
        std::memcpy(out128, &id, sizeof(id));
    });
}

int dgkr_comm_create_nccl(dgkr_ctx* ctx, const std::uint8_t* uid128, int rank, int world, dgkr_comm** out) {
    return guard([&] {
        if (!g_nccl.load()) fail(DGKR_COMM_ERROR, "libnccl.so.2 not found");
        if (world < 1 || rank < 0 || rank >= world) fail(DGKR_INVALID_ARGUMENT, "bad rank / world");
        if (world > kMaxCommWorld) fail(DGKR_INVALID_ARGUMENT, "world larger than the round-sum gather buffer");
        CK(cudaSetDevice(ctx->device));
        auto c = std::make_unique<NcclComm>();
        c->rank = rank;
        c->world = world;
        ncclUniqueId id;
        std::memcpy(&id, uid128, sizeof(id));
        NCK(g_nccl.commInitRank(&c->comm, world, id, rank));
        *out = c.release();
    });
}

void dgkr_comm_destroy(dgkr_comm* c) { delete c; }

int dgkr_comm_create_shm(dgkr_ctx* ctx, const char* name, int rank, int world, std::size_t slot_bytes,
                         dgkr_comm** out) {
    return guard([&] {
        if (world < 1 || rank < 0 || rank >= world) fail(DGKR_INVALID_ARGUMENT, "bad rank / world");
        if (world > kMaxCommWorld) fail(DGKR_INVALID_ARGUMENT, "world larger than the round-sum gather buffer");
        if (!name || name[0] != '/') fail(DGKR_INVALID_ARGUMENT, "shm name must start with '/'");
        auto c = std::make_unique<ShmComm>();
        c->rank = rank;
        c->world = world;
        c->name = name;
        c->owner = rank == 0;
        const std::size_t hb = 64;
        c->map_bytes = hb + static_cast<std::size_t>(world) * slot_bytes;
        const int fd = shm_open(name, O_CREAT | O_RDWR, 0600);
        if (fd < 0) fail(DGKR_COMM_ERROR, std::string("shm_open failed: ") + name);
        if (ftruncate(fd, static_cast<off_t>(c->map_bytes)) != 0) {
            close(fd);
            fail(DGKR_COMM_ERROR, "ftruncate failed");
        }
        void* p = mmap(nullptr, c->map_bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
        close(fd);
        if (p == MAP_FAILED) fail(DGKR_COMM_ERROR, "mmap failed");
        c->hdr = static_cast<ShmHeader*>(p);
        c->hdr->world = static_cast<std::uint32_t>(world);
        c->hdr->slot_bytes = slot_bytes;
        c->data = static_cast<std::uint8_t*>(p) + hb;
        if (ctx) {  // device exchanges need the pinned bounce buffer; host-only test comms do not
            CK(cudaSetDevice(ctx->device));
            CK(cudaMallocHost(reinterpret_cast<void**>(&c->bounce), std::max<std::size_t>(slot_bytes, 64)));
        }
        // not cudaHostRegister'ed: ranks sharing one GPU would register the same
        // physical pages twice, which corrupted device state (measured with 8 lanes x 2 ranks)
        (void)ctx;
        *out = c.release();
    });
}

int dgkr_comm_allgather_host(dgkr_comm* comm, const void* in, std::size_t bytes, void* out) {
    return guard([&] {
        auto* s = dynamic_cast<ShmComm*>(comm);
        if (!s) fail(DGKR_UNSUPPORTED, "host all-gather is a shared-memory communicator test hook");
        s->allgather_host(in, bytes, out);
    });
}

