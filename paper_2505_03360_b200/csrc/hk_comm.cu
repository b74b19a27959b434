// hk_comm.cu — NCCL communicator of a context: x-slab halo exchange and the
// driver's scalar all-reduces, C-ABI side.
//
// NCCL is resolved at run time (dlopen "libnccl.so.2"): inside a PyTorch
// process this is the NCCL torch already loaded, in a plain C++ caller the
// system one; nothing links against it, so loading the library never needs
// NCCL.  One communicator per context (= per GPU / rank); every call is
// stream-ordered on the context's stream.
//
// Halo contract (replaces the reference's in-process neighbour reads of
// kinetic_transport_rhs_periodic, src/transport.cpp:51-66, across ranks):
// slab f [ny][nx_local][n^3]; left halo = the left neighbour's last two
// columns, right halo = the right neighbour's first two, [ny][2][n^3] each,
// periodic over ranks (rank +- 1 mod nranks; one rank wraps onto itself).
#include <cuda.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>

#include "hk_internal.h"

namespace hk {
namespace {

struct NcclApi {
    bool loaded = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
#define HK_SYM(field, name) a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, name))
        HK_SYM(GetUniqueId, "ncclGetUniqueId");
        HK_SYM(CommInitRank, "ncclCommInitRank");
        HK_SYM(CommDestroy, "ncclCommDestroy");
        HK_SYM(GroupStart, "ncclGroupStart");
        HK_SYM(GroupEnd, "ncclGroupEnd");
        HK_SYM(Send, "ncclSend");
        HK_SYM(Recv, "ncclRecv");
        HK_SYM(AllReduce, "ncclAllReduce");
        HK_SYM(GetErrorString, "ncclGetErrorString");
#undef HK_SYM
        a.loaded = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.GroupStart && a.GroupEnd && a.Send &&
                   a.Recv && a.AllReduce && a.GetErrorString;
        return a;
    }();
    return api;
}

int check_nccl(hk_ctx ctx, ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return HK_OK;
    return fail(ctx, HK_NCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

}  // namespace

void comm_destroy(hk_ctx ctx) {
    if (ctx && ctx->comm && nccl().loaded) nccl().CommDestroy(static_cast<ncclComm_t>(ctx->comm));
    if (ctx) ctx->comm = nullptr;
}

int halo_columns_padded(hk_ctx ctx, const void* src, size_t cb, int64_t nx, int64_t ny, int w, void* pad) {
    const char* s = static_cast<const char*>(src);
    char* d = static_cast<char*>(pad);
    const size_t row = size_t(nx) * cb, prow = size_t(nx + 2 * w) * cb, wb = size_t(w) * cb;
    if (!ctx->comm || ctx->nranks < 2) {  // the slab is its own periodic neighbour
        int st = check_cuda(ctx, cudaMemcpy2DAsync(d, prow, s + row - wb, row, wb, ny, cudaMemcpyDeviceToDevice, ctx->stream),
                            "slab halo copy");
        if (!st)
            st = check_cuda(ctx, cudaMemcpy2DAsync(d + wb + row, prow, s, row, wb, ny, cudaMemcpyDeviceToDevice, ctx->stream),
                            "slab halo copy");
        return st;
    }
    if (!nccl().loaded) return fail(ctx, HK_NCCL, "libnccl.so.2 not found");
    const int left = (ctx->rank - 1 + ctx->nranks) % ctx->nranks, right = (ctx->rank + 1) % ctx->nranks;
    auto comm = static_cast<ncclComm_t>(ctx->comm);
    auto& api = nccl();
    int st = check_nccl(ctx, api.GroupStart(), "ncclGroupStart");
    if (st) return st;
    // same posting order as hk_halo_exchange: to the left, to the right, from the right, from the left
    for (int64_t j = 0; j < ny && !st; ++j)
        st = check_nccl(ctx, api.Send(s + j * row, wb, ncclInt8, left, comm, ctx->stream), "ncclSend");
    for (int64_t j = 0; j < ny && !st; ++j)
        st = check_nccl(ctx, api.Send(s + j * row + row - wb, wb, ncclInt8, right, comm, ctx->stream), "ncclSend");
    for (int64_t j = 0; j < ny && !st; ++j)
        st = check_nccl(ctx, api.Recv(d + j * prow + wb + row, wb, ncclInt8, right, comm, ctx->stream), "ncclRecv");
    for (int64_t j = 0; j < ny && !st; ++j)
        st = check_nccl(ctx, api.Recv(d + j * prow, wb, ncclInt8, left, comm, ctx->stream), "ncclRecv");
    const int st2 = check_nccl(ctx, api.GroupEnd(), "ncclGroupEnd");
    return st ? st : st2;
}

}  // namespace hk

using namespace hk;

extern "C" {

int hk_comm_unique_id(void* id_out) {
    if (!id_out) return HK_CONTRACT;
    if (!nccl().loaded) return HK_NCCL;
    ncclUniqueId id;
    if (nccl().GetUniqueId(&id) != ncclSuccess) return HK_NCCL;
    std::memcpy(id_out, &id, sizeof id);
    return HK_OK;
}

int hk_ctx_comm_init(hk_ctx ctx, int nranks, int rank, const void* id) {
    if (!ctx || !id || nranks < 1 || rank < 0 || rank >= nranks) return fail(ctx, HK_CONTRACT, "hk_ctx_comm_init: bad arguments");
    if (!nccl().loaded) return fail(ctx, HK_NCCL, "libnccl.so.2 not found");
    cudaSetDevice(ctx->device);
    comm_destroy(ctx);
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof uid);
    ncclComm_t c = nullptr;
    int st = check_nccl(ctx, nccl().CommInitRank(&c, nranks, uid, rank), "ncclCommInitRank");
    if (st) return st;
    ctx->comm = c;
    ctx->nranks = nranks;
    ctx->rank = rank;
    return HK_OK;
}

int hk_halo_exchange(hk_ctx ctx, int n, const double* f_dev, int64_t nx_local, int64_t ny, double* left_dev,
                     double* right_dev) {
    HK_RANGE("hk_halo_exchange");
    if (!ctx->comm) return fail(ctx, HK_CONTRACT, "hk_halo_exchange: context has no communicator (hk_ctx_comm_init)");
    if (n < 2 || nx_local < 2 || ny < 1 || !f_dev || !left_dev || !right_dev)
        return fail(ctx, HK_CONTRACT, "hk_halo_exchange: need nx_local >= 2 columns and non-null buffers");
    cudaSetDevice(ctx->device);
    const size_t nb = size_t(n) * n * n, blk = 2 * nb;  // two cells of one row
    const int left = (ctx->rank - 1 + ctx->nranks) % ctx->nranks, right = (ctx->rank + 1) % ctx->nranks;
    auto comm = static_cast<ncclComm_t>(ctx->comm);
    auto& api = nccl();
    int st = check_nccl(ctx, api.GroupStart(), "ncclGroupStart");
    if (st) return st;
    // Per peer pair, matching is in posting order: all "to the left" sends,
    // then all "to the right"; receives "from the right" first, then "from
    // the left" (correct for 1, 2 and >2 ranks alike).
    for (int64_t j = 0; j < ny && !st; ++j)
        st = check_nccl(ctx, api.Send(f_dev + (size_t)j * nx_local * nb, blk, ncclFloat64, left, comm, ctx->stream), "ncclSend");
    for (int64_t j = 0; j < ny && !st; ++j)
        st = check_nccl(ctx, api.Send(f_dev + ((size_t)j * nx_local + nx_local - 2) * nb, blk, ncclFloat64, right, comm, ctx->stream),
                        "ncclSend");
    for (int64_t j = 0; j < ny && !st; ++j)
        st = check_nccl(ctx, api.Recv(right_dev + (size_t)j * blk, blk, ncclFloat64, right, comm, ctx->stream), "ncclRecv");
    for (int64_t j = 0; j < ny && !st; ++j)
        st = check_nccl(ctx, api.Recv(left_dev + (size_t)j * blk, blk, ncclFloat64, left, comm, ctx->stream), "ncclRecv");
    const int st2 = check_nccl(ctx, api.GroupEnd(), "ncclGroupEnd");
    return st ? st : st2;
}

int hk_allreduce_scalars(hk_ctx ctx, double* buf_dev, int64_t count, int op) {
    HK_RANGE("hk_allreduce_scalars");
    if (!ctx->comm) return fail(ctx, HK_CONTRACT, "hk_allreduce_scalars: context has no communicator");
    if (count < 0 || (count > 0 && !buf_dev)) return fail(ctx, HK_CONTRACT, "hk_allreduce_scalars: bad buffer");
    if (op != HK_REDUCE_SUM && op != HK_REDUCE_MAX) return fail(ctx, HK_CONTRACT, "hk_allreduce_scalars: op must be SUM or MAX");
    if (count == 0) return HK_OK;
    cudaSetDevice(ctx->device);
    return check_nccl(ctx,
                      nccl().AllReduce(buf_dev, buf_dev, (size_t)count, ncclFloat64, op == HK_REDUCE_SUM ? ncclSum : ncclMax,
                                       static_cast<ncclComm_t>(ctx->comm), ctx->stream),
                      "ncclAllReduce");
}

// ---- CUDA IPC: another rank's device buffer mapped into this process ----
// A handle names the whole allocation; a pointer inside a sub-allocating pool
// (PyTorch's caching allocator) also needs its offset from the allocation base
// (driver cuMemGetAddressRange, resolved through the runtime's entry points).
int hk_ipc_handle(hk_ctx ctx, const void* dev_ptr, void* handle_out, int64_t* offset_out) {
    if (!dev_ptr || !handle_out) return fail(ctx, HK_CONTRACT, "hk_ipc_handle: null pointer");
    cudaSetDevice(ctx->device);
    cudaIpcMemHandle_t h;
    int st = check_cuda(ctx, cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)), "cudaIpcGetMemHandle");
    if (st) return st;
    std::memcpy(handle_out, &h, sizeof h);
    if (offset_out) {
        using Pfn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
        static Pfn range = nullptr;
        if (!range) {
            void* fn = nullptr;
            cudaDriverEntryPointQueryResult q;
            if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
                q != cudaDriverEntryPointSuccess || !fn)
                return fail(ctx, HK_CUDA, "cuMemGetAddressRange unavailable");
            range = reinterpret_cast<Pfn>(fn);
        }
        CUdeviceptr base = 0;
        size_t size = 0;
        if (range(&base, &size, (CUdeviceptr)dev_ptr) != CUDA_SUCCESS) return fail(ctx, HK_CUDA, "cuMemGetAddressRange");
        *offset_out = (int64_t)((CUdeviceptr)dev_ptr - base);
    }
    return HK_OK;
}

int hk_ipc_open(hk_ctx ctx, const void* handle, void** dev_ptr_out) {
    if (!handle || !dev_ptr_out) return fail(ctx, HK_CONTRACT, "hk_ipc_open: null pointer");
    cudaSetDevice(ctx->device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof h);
    return check_cuda(ctx, cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
}

int hk_ipc_close(hk_ctx ctx, void* dev_ptr) {
    cudaSetDevice(ctx->device);
    return check_cuda(ctx, cudaIpcCloseMemHandle(dev_ptr), "cudaIpcCloseMemHandle");
}

int hk_ctx_comm_info(hk_ctx ctx, int* nranks, int* rank) {
    if (nranks) *nranks = ctx->comm ? ctx->nranks : 0;
    if (rank) *rank = ctx->comm ? ctx->rank : -1;
    return HK_OK;
}

}  // extern "C"
