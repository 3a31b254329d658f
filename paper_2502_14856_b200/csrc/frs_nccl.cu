// The vocab-parallel verify head's exchange on the C ABI (SURVEY.md §8(b) frs_allgather_merge,
// §8(e) row 3): each rank runs K3 on its contiguous vocabulary shard (ids offset by the shard
// start), NCCL all-gathers the per-row (value, id) pairs of every rank over NVLink / NVSwitch, and
// K5 merges them by (value desc, id asc) — argmax's strict '>' over ascending ids
// (kernels.cpp:113-122) — all stream-ordered on the caller's stream. The reference has no
// multi-GPU path (it is a single-threaded CPU library); this is the sharded form of its argmax.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2; the copy already loaded in the process,
// e.g. torch's, is reused), so the library has no link-time NCCL dependency. Failures return
// FRS_ENCCL with ncclGetErrorString's text; ncclCommGetAsyncError is checked after every call.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>

#include "frs_common.cuh"

namespace frs {
namespace {

struct NcclApi {
    ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*commCount)(const ncclComm_t, int *) = nullptr;
    ncclResult_t (*commUserRank)(const ncclComm_t, int *) = nullptr;
    ncclResult_t (*commGetAsyncError)(ncclComm_t, ncclResult_t *) = nullptr;
    ncclResult_t (*allGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    const char *(*getErrorString)(ncclResult_t) = nullptr;
    bool ok = false;
    std::string why;
};

const NcclApi &nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's copy (torch's)
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = "libnccl.so.2 not found";
            return;
        }
        auto sym = [&](auto &fp, const char *name) {
            fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
            return fp != nullptr;
        };
        api.ok = sym(api.getUniqueId, "ncclGetUniqueId") && sym(api.commInitRank, "ncclCommInitRank") &&
                 sym(api.commDestroy, "ncclCommDestroy") && sym(api.commCount, "ncclCommCount") &&
                 sym(api.commUserRank, "ncclCommUserRank") && sym(api.commGetAsyncError, "ncclCommGetAsyncError") &&
                 sym(api.allGather, "ncclAllGather") && sym(api.groupStart, "ncclGroupStart") &&
                 sym(api.groupEnd, "ncclGroupEnd") && sym(api.getErrorString, "ncclGetErrorString");
        if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
    });
    return api;
}

int nccl_fail(ncclResult_t r, const char *what) {
    const NcclApi &n = nccl();
    return fail(FRS_ENCCL, std::string(what) + ": " + (n.getErrorString ? n.getErrorString(r) : "nccl error"));
}

#define FRS_NCCL_TRY(expr, what)                             \
    do {                                                     \
        const ncclResult_t r_ = (expr);                      \
        if (r_ != ncclSuccess) return nccl_fail(r_, (what)); \
    } while (0)

int async_check(ncclComm_t comm) {
    ncclResult_t a = ncclSuccess;
    FRS_NCCL_TRY(nccl().commGetAsyncError(comm, &a), "ncclCommGetAsyncError");
    if (a != ncclSuccess && a != ncclInProgress) return nccl_fail(a, "NCCL communicator (async)");
    return FRS_OK;
}

}  // namespace
}  // namespace frs

using namespace frs;

extern "C" {

int frs_nccl_get_unique_id(void *id_out) {
    FRS_REQUIRE(id_out, "nccl: null pointer");
    const NcclApi &n = nccl();
    if (!n.ok) return fail(FRS_ENCCL, "NCCL unavailable: " + n.why);
    ncclUniqueId id;
    FRS_NCCL_TRY(n.getUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(id_out, &id, sizeof(id));
    return FRS_OK;
}

int frs_nccl_comm_init(frs_ctx *ctx, int nranks, const void *id, int rank, void **comm_out) {
    FRS_REQUIRE(ctx && id && comm_out, "nccl: null pointer");
    FRS_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "nccl: rank out of range");
    const NcclApi &n = nccl();
    if (!n.ok) return fail(FRS_ENCCL, "NCCL unavailable: " + n.why);
    FRS_CUDA_TRY(cudaSetDevice(ctx->device));
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    ncclComm_t comm = nullptr;
    FRS_NCCL_TRY(n.commInitRank(&comm, nranks, uid, rank), "ncclCommInitRank");
    *comm_out = comm;
    return FRS_OK;
}

int frs_nccl_comm_destroy(void *comm) {
    if (!comm) return FRS_OK;
    const NcclApi &n = nccl();
    if (!n.ok) return fail(FRS_ENCCL, "NCCL unavailable: " + n.why);
    FRS_NCCL_TRY(n.commDestroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy");
    return FRS_OK;
}

int frs_verify_head_argmax_vp(frs_ctx *ctx, void *comm_v, const float *h, int m, int d, const void *W_shard,
                              int v_rows, int w_dtype, int32_t id_offset, int mode, int32_t *out_id, float *out_val,
                              uint32_t *out_flags, void *stream) {
    FRS_REQUIRE(ctx && comm_v && out_id && out_val, "verify (vocab-parallel): null pointer");
    const NcclApi &n = nccl();
    if (!n.ok) return fail(FRS_ENCCL, "NCCL unavailable: " + n.why);
    ncclComm_t comm = static_cast<ncclComm_t>(comm_v);
    int world = 0, rank = 0, st;
    FRS_NCCL_TRY(n.commCount(comm, &world), "ncclCommCount");
    FRS_NCCL_TRY(n.commUserRank(comm, &rank), "ncclCommUserRank");
    if ((st = async_check(comm))) return st;
    // this rank's pairs, then every rank's: [world][m] values | [world][m] ids
    const size_t need = (size_t)m * 8 + (size_t)world * m * 8;
    if ((st = ctx->vp_buf.ensure(need))) return st;
    float *my_val = static_cast<float *>(ctx->vp_buf.ptr);
    int32_t *my_id = reinterpret_cast<int32_t *>(my_val + m);
    float *all_val = reinterpret_cast<float *>(my_id + m);
    int32_t *all_id = reinterpret_cast<int32_t *>(all_val + (size_t)world * m);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if ((st = frs_verify_head_argmax(ctx, h, m, d, W_shard, v_rows, w_dtype, id_offset, mode, my_id, my_val, out_flags,
                                     stream)))
        return st;
    FRS_NCCL_TRY(n.groupStart(), "ncclGroupStart");
    ncclResult_t r1 = n.allGather(my_val, all_val, (size_t)m, ncclFloat32, comm, s);
    ncclResult_t r2 = n.allGather(my_id, all_id, (size_t)m, ncclInt32, comm, s);
    ncclResult_t r3 = n.groupEnd();
    if (r1 != ncclSuccess) return nccl_fail(r1, "ncclAllGather (values)");
    if (r2 != ncclSuccess) return nccl_fail(r2, "ncclAllGather (ids)");
    if (r3 != ncclSuccess) return nccl_fail(r3, "ncclGroupEnd");
    if ((st = async_check(comm))) return st;
    (void)rank;
    return frs_argmax_merge(ctx, all_val, all_id, world, m, out_val, out_id, stream);
}

}  // extern "C"
