// probe.cu — bandwidth probe for the second roofline ("measure L2
// read bandwidth on the box with a repeated read of a buffer of ~1/4 of L2").
// A persistent grid (one wave: 148 SMs x 4 CTAs of 512 threads) streams the
// buffer `reps` times with 128-bit loads, 4 independent loads in flight per
// thread, and folds the values into one word per CTA (so no load is dead).
// Working sets well under the 126 MB L2 measure L2 read bandwidth after the
// first pass; larger ones measure HBM.
#include "dr_internal.h"

namespace dr {
namespace {

__global__ void __launch_bounds__(512) probe_read_kernel(const float4 *__restrict__ buf, int64_t n4,
                                                         int reps, float *__restrict__ sink) {
    float acc = 0.f;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; ++r) {
        int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        for (; i + 3 * stride < n4; i += 4 * stride) {
            const float4 a = __ldcg(buf + i), b = __ldcg(buf + i + stride);
            const float4 c = __ldcg(buf + i + 2 * stride), d = __ldcg(buf + i + 3 * stride);
            acc += (a.x + b.y) + (c.z + d.w);
        }
        for (; i < n4; i += stride) acc += __ldcg(buf + i).x;
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 16);
    if (threadIdx.x == 0) sink[blockIdx.x] = acc;
}

}  // namespace
}  // namespace dr

using namespace dr;

extern "C" dr_status dr_probe_read(const void *buf, int64_t bytes, int32_t reps, float *sink,
                                   void *stream) {
    clear_error();
    try {
        DR_CHECK(buf && sink && bytes >= 16 && reps >= 1, DR_ERR_INVALID_ARGUMENT, "probe_read: bad args");
        DR_CHECK((reinterpret_cast<uintptr_t>(buf) & 15) == 0, DR_ERR_INVALID_ARGUMENT,
                 "probe_read: buffer not 16-B aligned");
        probe_read_kernel<<<148 * 4, 512, 0, (cudaStream_t)stream>>>(
            reinterpret_cast<const float4 *>(buf), bytes / 16, reps, sink);
        note_launch("probe_read");
        return DR_OK;
    } catch (const Error &e) {
        set_error(e.status, e.msg);
        return e.status;
    }
}
