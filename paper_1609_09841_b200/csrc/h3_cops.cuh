// Constant-bank operator ring for the DFMA kernels (include from ONE translation unit).
//
// Device side: cop<OFF>() reads h3_cop[OFF] with an immediate-address `ld.const` in a volatile
// asm, so the front end cannot hoist it out of the plane loop into registers; ptxas turns it
// into a constant/uniform-register operand of the consuming DFMA.  sfor<K>(f) unrolls f over
// std::integral_constant<int, 0..K-1> so operator offsets are compile-time constants.
//
// Host side: cop_acquire() returns a slot holding the requested operator set (uploading it with
// cudaMemcpyToSymbolAsync on the caller's stream when no slot matches, then recording the slot's
// `ready` event; a caller on another stream that finds the slot waits on that event);
// cop_release() records the launch's completion event on the slot.  A slot is overwritten only
// after every recorded user has completed (the uploading stream waits on their events), and never
// while a caller holds it between acquire and release (its launch is not recorded yet): such
// slots are skipped, and if all are held the caller waits for one to be released.
#pragma once
#include <cuda_runtime.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <type_traits>
#include <utility>
#include <vector>

namespace h3 {

constexpr int COP_SLOTS = 4;
constexpr int COP_SLOT = 512;  // doubles per slot (4 KB); 16 KB of the 64 KB constant space

}  // namespace h3

// global scope, unmangled: the PTX name `h3_cop` is used in the ld.const asm below
__constant__ double h3_cop[h3::COP_SLOTS * h3::COP_SLOT];

namespace h3 {

template <int OFF>
__device__ __forceinline__ double cop() {
    static_assert(OFF >= 0 && OFF < COP_SLOTS * COP_SLOT, "constant operator offset out of range");
    double v;
    asm volatile("ld.const.f64 %0, [h3_cop+%1];" : "=d"(v) : "n"(OFF * 8));
    return v;
}

template <class F, int... Is>
__device__ __forceinline__ void sfor_impl(F&& f, std::integer_sequence<int, Is...>) {
    (f(std::integral_constant<int, Is>{}), ...);
}
template <int K, class F>
__device__ __forceinline__ void sfor(F&& f) {
    sfor_impl(f, std::make_integer_sequence<int, K>{});
}

// ---- host ring ------------------------------------------------------------------------------
struct CopSlotState {
    int count = -1;
    double bits[COP_SLOT];
    std::vector<cudaEvent_t> users;
    cudaEvent_t ready = nullptr;  // recorded after the upload; other streams wait on it
    int held = 0;                 // callers between cop_acquire and cop_release
};
struct CopDeviceState {
    CopSlotState slot[COP_SLOTS];
    int next = 0;
};
constexpr int COP_MAX_DEVICES = 64;

static std::mutex& cop_mutex() {
    static std::mutex m;
    return m;
}
static std::condition_variable& cop_released() {
    static std::condition_variable cv;
    return cv;
}
static CopDeviceState& cop_device(int dev) {
    static CopDeviceState states[COP_MAX_DEVICES];
    return states[dev];
}

// 0 on success (slot in *slot), else a cudaError_t.
static int cop_acquire(const double* ops, int count, cudaStream_t st, int* slot) {
    if (count < 1 || count > COP_SLOT) return (int)cudaErrorInvalidValue;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return (int)e;
    if (dev < 0 || dev >= COP_MAX_DEVICES) return (int)cudaErrorInvalidDevice;
    std::unique_lock<std::mutex> lk(cop_mutex());
    CopDeviceState& D = cop_device(dev);
    for (int s = 0; s < COP_SLOTS; ++s)
        if (D.slot[s].count == count && std::memcmp(D.slot[s].bits, ops, count * sizeof(double)) == 0) {
            // the upload may still be queued on another stream: order this stream after it
            if (D.slot[s].ready) {
                e = cudaStreamWaitEvent(st, D.slot[s].ready, 0);
                if (e != cudaSuccess) return (int)e;
            }
            ++D.slot[s].held;
            *slot = s;
            return 0;
        }
    int s = -1;
    for (;;) {  // next slot in ring order that no caller holds
        for (int i = 0; i < COP_SLOTS && s < 0; ++i) {
            const int c = (D.next + i) % COP_SLOTS;
            if (D.slot[c].held == 0) s = c;
        }
        if (s >= 0) break;
        cop_released().wait(lk);  // all COP_SLOTS held by concurrent callers: wait for a release
    }
    D.next = (s + 1) % COP_SLOTS;
    CopSlotState& S = D.slot[s];
    for (cudaEvent_t ev : S.users) {
        e = cudaStreamWaitEvent(st, ev, 0);
        cudaEventDestroy(ev);
        if (e != cudaSuccess) return (int)e;
    }
    S.users.clear();
    S.count = -1;
    e = cudaMemcpyToSymbolAsync(h3_cop, ops, count * sizeof(double), (size_t)s * COP_SLOT * sizeof(double),
                                cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return (int)e;
    if (!S.ready) {
        e = cudaEventCreateWithFlags(&S.ready, cudaEventDisableTiming);
        if (e != cudaSuccess) return (int)e;
    }
    e = cudaEventRecord(S.ready, st);
    if (e != cudaSuccess) return (int)e;
    std::memcpy(S.bits, ops, count * sizeof(double));
    S.count = count;
    ++S.held;
    *slot = s;
    return 0;
}

static int cop_release(int slot, cudaStream_t st) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return (int)e;
    std::lock_guard<std::mutex> lk(cop_mutex());
    CopSlotState& S = cop_device(dev).slot[slot];
    if (S.held > 0 && --S.held == 0) cop_released().notify_all();
    // drop completed users so the list stays short
    size_t keep = 0;
    for (size_t i = 0; i < S.users.size(); ++i) {
        if (cudaEventQuery(S.users[i]) == cudaSuccess) cudaEventDestroy(S.users[i]);
        else S.users[keep++] = S.users[i];
    }
    S.users.resize(keep);
    cudaEvent_t ev;
    e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return (int)e;
    e = cudaEventRecord(ev, st);
    if (e != cudaSuccess) {
        cudaEventDestroy(ev);
        return (int)e;
    }
    S.users.push_back(ev);
    return 0;
}

}  // namespace h3

