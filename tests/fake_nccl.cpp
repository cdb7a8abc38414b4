// Test infrastructure: a minimal NCCL stand-in so the multi-process sharded
// path (shard.cu: ncclCommInitRank, ncclAllGather, ncclBroadcast and the
// CUDA IPC pulls between ranks) can run as several processes on ONE GPU —
// real NCCL refuses two ranks on one device. Collectives are synchronous on
// the host (the stream is drained first) and exchange their bytes through a
// POSIX shared-memory segment named in the unique id (unique per run: a
// reused segment would carry stale barrier counters). Send/Recv are not
// provided (the shards' NVLink pull does not use them). Loaded through
// ETWG_NCCL_LIB by tests/test_gpu_multiprocess.py; never part of the product.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <ctime>

extern "C" {

typedef struct {
    char internal[128];
} ncclUniqueId;
typedef enum { ncclSuccess = 0, ncclUnhandledCudaError = 1, ncclSystemError = 2, ncclInternalError = 3,
               ncclInvalidArgument = 4, ncclInvalidUsage = 5 } ncclResult_t;
typedef int ncclDataType_t;  // only byte counts are used (ncclUint8)

constexpr size_t kSlot = 1 << 16;
constexpr int kMaxRanks = 8;

struct Shm {
    std::atomic<int> arrived;
    std::atomic<int> generation;
    char pad[56];
    char slot[kMaxRanks][kSlot];
};

struct Comm {
    int rank, nranks;
    Shm* shm;
    char name[128];
};
typedef Comm* ncclComm_t;

static void barrier(Comm* c) {
    const int gen = c->shm->generation.load();
    if (c->shm->arrived.fetch_add(1) + 1 == c->nranks) {
        c->shm->arrived.store(0);
        c->shm->generation.fetch_add(1);
    } else {
        while (c->shm->generation.load() == gen) usleep(20);
    }
}

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
    std::memset(id, 0, sizeof *id);
    timespec ts;
    clock_gettime(CLOCK_REALTIME, &ts);
    std::snprintf(id->internal, sizeof id->internal, "/fakenccl_%d_%ld_%ld", static_cast<int>(getpid()),
                  static_cast<long>(ts.tv_sec), static_cast<long>(ts.tv_nsec));
    return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
    if (nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks) return ncclInvalidArgument;
    const int fd = shm_open(id.internal, O_CREAT | O_RDWR, 0600);
    if (fd < 0) return ncclSystemError;
    if (ftruncate(fd, sizeof(Shm)) != 0) return ncclSystemError;
    void* p = mmap(nullptr, sizeof(Shm), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) return ncclSystemError;
    Comm* c = new Comm{rank, nranks, static_cast<Shm*>(p), {}};
    std::memcpy(c->name, id.internal, sizeof c->name);
    barrier(c);
    *comm = c;
    return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) {
    if (!comm) return ncclSuccess;
    barrier(comm);
    munmap(comm->shm, sizeof(Shm));
    if (comm->rank == 0) shm_unlink(comm->name);
    delete comm;
    return ncclSuccess;
}

// Copies go on the caller's stream and are drained there: a pageable-host
// cudaMemcpy can return before its DMA lands, and the caller's (non-blocking)
// stream would then read stale device memory.
static bool d2h(void* dst, const void* src, size_t n, cudaStream_t st) {
    return cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, st) == cudaSuccess &&
           cudaStreamSynchronize(st) == cudaSuccess;
}
static bool h2d(void* dst, const void* src, size_t n, cudaStream_t st) {
    return cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, st) == cudaSuccess &&
           cudaStreamSynchronize(st) == cudaSuccess;
}

ncclResult_t ncclAllGather(const void* send, void* recv, size_t count, ncclDataType_t, ncclComm_t c,
                           cudaStream_t stream) {
    if (count > kSlot) return ncclInvalidUsage;
    if (cudaStreamSynchronize(stream) != cudaSuccess) return ncclUnhandledCudaError;
    if (!d2h(c->shm->slot[c->rank], send, count, stream)) return ncclUnhandledCudaError;
    barrier(c);
    for (int r = 0; r < c->nranks; ++r)
        if (!h2d(static_cast<char*>(recv) + r * count, c->shm->slot[r], count, stream)) return ncclUnhandledCudaError;
    barrier(c);
    return ncclSuccess;
}

ncclResult_t ncclBroadcast(const void* send, void* recv, size_t count, ncclDataType_t, int root, ncclComm_t c,
                           cudaStream_t stream) {
    if (count > kSlot) return ncclInvalidUsage;
    if (cudaStreamSynchronize(stream) != cudaSuccess) return ncclUnhandledCudaError;
    if (c->rank == root && !d2h(c->shm->slot[0], send, count, stream)) return ncclUnhandledCudaError;
    barrier(c);
    if (!h2d(recv, c->shm->slot[0], count, stream)) return ncclUnhandledCudaError;
    barrier(c);
    return ncclSuccess;
}

ncclResult_t ncclSend(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) { return ncclInvalidUsage; }
ncclResult_t ncclRecv(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) { return ncclInvalidUsage; }
ncclResult_t ncclGroupStart() { return ncclSuccess; }
ncclResult_t ncclGroupEnd() { return ncclSuccess; }

const char* ncclGetErrorString(ncclResult_t r) {
    switch (r) {
        case ncclSuccess: return "success (fake nccl)";
        case ncclInvalidUsage: return "invalid usage (fake nccl: send/recv and messages > 64 KiB unsupported)";
        default: return "error (fake nccl)";
    }
}
}
