// Multi-GPU plumbing: NCCL loaded at run time (dlopen, so libcfpq loads on hosts without
// NCCL), row-block partitions of the bit matrices, and the per-iteration exchange of the
// dense engine (in-place all-gather of every rank's row block of T_k + all-reduce of the
// new-cell count = the "changed" flag of Alg. 1 line 8).
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

#include "cfpq_internal.cuh"

namespace cfpq {

struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;   // NCCL >= 2.18
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi g_nccl;
static std::mutex g_nccl_mu;

static bool load_nccl(std::string* err) {
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    if (g_nccl.h) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    void* h = nullptr;
    for (const char* nm : names)
        if ((h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) {
        if (err) *err = std::string("cannot dlopen libnccl.so.2: ") + dlerror();
        return false;
    }
#define SYM(f)                                                                      \
    g_nccl.f = reinterpret_cast<decltype(g_nccl.f)>(dlsym(h, "nccl" #f));           \
    if (!g_nccl.f) {                                                                \
        if (err) *err = "libnccl lacks nccl" #f;                                    \
        dlclose(h);                                                                 \
        return false;                                                               \
    }
    SYM(GetUniqueId);
    SYM(CommInitRank);
    SYM(AllGather);
    SYM(AllReduce);
    SYM(GroupStart);
    SYM(GroupEnd);
    SYM(CommDestroy);
    SYM(GetErrorString);
#undef SYM
    g_nccl.CommSplit = reinterpret_cast<decltype(g_nccl.CommSplit)>(dlsym(h, "ncclCommSplit"));
    g_nccl.h = h;
    return true;
}

bool nccl_unique_id(void* out, std::string* err) {
    if (!load_nccl(err)) return false;
    ncclUniqueId id;
    ncclResult_t r = g_nccl.GetUniqueId(&id);
    if (r != ncclSuccess) {
        if (err) *err = std::string("ncclGetUniqueId: ") + g_nccl.GetErrorString(r);
        return false;
    }
    memcpy(out, &id, sizeof(id));
    return true;
}

size_t nccl_unique_id_bytes() { return sizeof(ncclUniqueId); }

void* nccl_comm_create(const void* id_bytes, int world, int rank, std::string* err) {
    if (!load_nccl(err)) return nullptr;
    ncclUniqueId id;
    memcpy(&id, id_bytes, sizeof(id));
    ncclComm_t comm = nullptr;
    ncclResult_t r = g_nccl.CommInitRank(&comm, world, id, rank);
    if (r != ncclSuccess) {
        if (err) *err = std::string("ncclCommInitRank: ") + g_nccl.GetErrorString(r);
        return nullptr;
    }
    return comm;
}

void nccl_comm_destroy(void* comm) {
    if (comm && g_nccl.h) g_nccl.CommDestroy((ncclComm_t)comm);
}

// In-place all-gather of equal row blocks of each matrix + sum of one uint64 counter.
bool nccl_exchange_rows(void* comm, uint32_t* const* mats, int n_mats, size_t block_words, int rank,
                        unsigned long long* counter, cudaStream_t s, std::string* err) {
    ncclComm_t c = (ncclComm_t)comm;
    ncclResult_t r = g_nccl.GroupStart();
    for (int q = 0; q < n_mats && r == ncclSuccess; ++q)
        r = g_nccl.AllGather(mats[q] + (size_t)rank * block_words, mats[q], block_words, ncclUint32, c, s);
    if (r == ncclSuccess && counter) r = g_nccl.AllReduce(counter, counter, 1, ncclUint64, ncclSum, c, s);
    ncclResult_t r2 = g_nccl.GroupEnd();
    if (r == ncclSuccess) r = r2;
    if (r != ncclSuccess) {
        if (err) *err = std::string("NCCL exchange: ") + g_nccl.GetErrorString(r);
        return false;
    }
    return true;
}

// In-place all-gather of `count` uint64 per rank: buf[rank*count, +count) -> every rank's
// buf[0, world*count).  Used by the sparse engine's Δ exchange (counts, then cells).
bool nccl_allgather_u64(void* comm, uint64_t* buf, size_t count, int rank, cudaStream_t s, std::string* err) {
    ncclResult_t r = g_nccl.AllGather(buf + (size_t)rank * count, buf, count, ncclUint64, (ncclComm_t)comm, s);
    if (r != ncclSuccess) {
        if (err) *err = std::string("NCCL all-gather: ") + g_nccl.GetErrorString(r);
        return false;
    }
    return true;
}

// Sub-communicator (2-D process grid rows / columns): ranks with the same color, ordered by key.
void* nccl_comm_split(void* comm, int color, int key, std::string* err) {
    if (!g_nccl.CommSplit) {
        if (err) *err = "libnccl lacks ncclCommSplit (NCCL >= 2.18 needed for 2-D grids)";
        return nullptr;
    }
    ncclComm_t out = nullptr;
    ncclResult_t r = g_nccl.CommSplit((ncclComm_t)comm, color, key, &out, nullptr);
    if (r != ncclSuccess) {
        if (err) *err = std::string("ncclCommSplit: ") + g_nccl.GetErrorString(r);
        return nullptr;
    }
    return out;
}

bool nccl_allgather_u32(void* comm, uint32_t* buf, size_t count, int rank, cudaStream_t s, std::string* err) {
    ncclResult_t r = g_nccl.AllGather(buf + (size_t)rank * count, buf, count, ncclUint32, (ncclComm_t)comm, s);
    if (r != ncclSuccess) {
        if (err) *err = std::string("NCCL all-gather: ") + g_nccl.GetErrorString(r);
        return false;
    }
    return true;
}

bool nccl_allreduce_sum_u64(void* comm, unsigned long long* buf, size_t count, cudaStream_t s, std::string* err) {
    ncclResult_t r = g_nccl.AllReduce(buf, buf, count, ncclUint64, ncclSum, (ncclComm_t)comm, s);
    if (r != ncclSuccess) {
        if (err) *err = std::string("NCCL all-reduce: ") + g_nccl.GetErrorString(r);
        return false;
    }
    return true;
}

bool nccl_group(bool start, std::string* err) {
    ncclResult_t r = start ? g_nccl.GroupStart() : g_nccl.GroupEnd();
    if (r != ncclSuccess) {
        if (err) *err = std::string("NCCL group: ") + g_nccl.GetErrorString(r);
        return false;
    }
    return true;
}

// 2-D grid: rows split like dense_partition over gr, 256-column tiles split over gc.
void dense_partition2(int64_t n, int gr, int gc, int a, int b, int64_t* ti_lo, int64_t* ti_hi, int64_t* tj_lo,
                      int64_t* tj_hi) {
    int64_t br;
    dense_partition(n, gr, a, ti_lo, ti_hi, &br);
    const int64_t np = ((n + 255) / 256) * 256;
    const int64_t jt = np / 256 > 0 ? np / 256 : 1;
    const int64_t bj = (jt + gc - 1) / gc;
    *tj_lo = std::min<int64_t>((int64_t)b * bj, jt);
    *tj_hi = std::min<int64_t>(*tj_lo + bj, jt);
}

// Row-block partition of the dense engine: tiles of 128 rows, equal blocks of
// ceil(tiles/world) tiles (the last ranks may own fewer or none).
void dense_partition(int64_t n, int world, int rank, int64_t* tile_lo, int64_t* tile_hi, int64_t* block_rows) {
    const int64_t np = ((n + 255) / 256) * 256;
    const int64_t tiles = np / 128 > 0 ? np / 128 : 1;
    const int64_t bt = (tiles + world - 1) / world;
    int64_t lo = std::min<int64_t>((int64_t)rank * bt, tiles), hi = std::min<int64_t>(lo + bt, tiles);
    *tile_lo = lo;
    *tile_hi = hi;
    *block_rows = bt * 128;
}

}  // namespace cfpq
