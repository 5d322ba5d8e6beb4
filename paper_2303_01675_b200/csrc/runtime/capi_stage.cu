// C-ABI over GptStage (include/ptk.h ptk_stage_*).  Exceptions never cross
// the boundary: they become a status code plus ptk_last_error().
#include <cstring>
#include <exception>

#include "../../../include/ptk.h"
#include "errors.h"
#include "gpt_stage.h"

#include "capi_handles.h"

namespace {

template <class F>
int guarded(const char* what, F&& f) {
    try {
        f();
        return PTK_OK;
    } catch (const std::exception& e) {
        return ptk::set_error(PTK_ERR_CUDA, std::string(what) + ": " + e.what());
    }
}

}  // namespace

extern "C" int ptk_stage_create(const ptk_gpt_config* cfg, ptk_stage** out) {
    if (cfg == nullptr || out == nullptr) return ptk::set_error(PTK_ERR_ARG, "ptk_stage_create: null argument");
    try {
        *out = new ptk_stage(new ptk::GptStage(*cfg), true);
        return PTK_OK;
    } catch (const std::invalid_argument& e) {
        return ptk::set_error(PTK_ERR_ARG, e.what());
    } catch (const std::exception& e) {
        return ptk::set_error(PTK_ERR_CUDA, e.what());
    }
}

extern "C" int ptk_stage_destroy(ptk_stage* st) {
    delete st;
    return PTK_OK;
}

extern "C" int ptk_stage_forward(ptk_stage* st, int slot, const int32_t* tok, const void* x_in, const int32_t* labels,
                                 void* x_out, void* stream) {
    if (!st) return ptk::set_error(PTK_ERR_ARG, "null stage");
    return guarded("ptk_stage_forward", [&] {
        st->impl->forward(slot, tok, static_cast<const __nv_bfloat16*>(x_in), labels, static_cast<__nv_bfloat16*>(x_out),
                         static_cast<cudaStream_t>(stream));
    });
}

extern "C" int ptk_stage_backward(ptk_stage* st, int slot, const int32_t* tok, const void* dy, void* dx,
                                  void* stream) {
    if (!st) return ptk::set_error(PTK_ERR_ARG, "null stage");
    return guarded("ptk_stage_backward", [&] {
        st->impl->backward(slot, tok, static_cast<const __nv_bfloat16*>(dy), static_cast<__nv_bfloat16*>(dx),
                          static_cast<cudaStream_t>(stream));
        st->impl->finalize_grads(static_cast<cudaStream_t>(stream));  // grads complete in stream order
    });
}

extern "C" int ptk_stage_optimizer_step(ptk_stage* st, float lr, float wd, void* stream) {
    if (!st) return ptk::set_error(PTK_ERR_ARG, "null stage");
    return guarded("ptk_stage_optimizer_step",
                   [&] { st->impl->optimizer_step(lr, wd, static_cast<cudaStream_t>(stream)); });
}

extern "C" int ptk_stage_zero_grads(ptk_stage* st, void* stream) {
    if (!st) return ptk::set_error(PTK_ERR_ARG, "null stage");
    return guarded("ptk_stage_zero_grads", [&] { st->impl->zero_grads(static_cast<cudaStream_t>(stream)); });
}

extern "C" int ptk_stage_buffers(ptk_stage* st, float** master, void** weights, float** grads, float** loss,
                                 int64_t* numel) {
    if (!st) return ptk::set_error(PTK_ERR_ARG, "null stage");
    if (master) *master = st->impl->master();
    if (weights) *weights = st->impl->weights();
    if (grads) *grads = st->impl->grads();
    if (loss) *loss = st->impl->loss_accumulator();
    if (numel) *numel = st->impl->param_count();
    return PTK_OK;
}

extern "C" int ptk_stage_param(ptk_stage* st, int i, char* name_buf, size_t cap, int64_t* offset, int64_t* rows,
                               int64_t* cols) {
    if (!st) return ptk::set_error(PTK_ERR_ARG, "null stage");
    const auto& ps = st->impl->params();
    if (i < 0 || static_cast<size_t>(i) >= ps.size()) return PTK_ERR_ARG;
    const ptk::ParamInfo& p = ps[static_cast<size_t>(i)];
    if (name_buf && cap) {
        std::strncpy(name_buf, p.name.c_str(), cap - 1);
        name_buf[cap - 1] = '\0';
    }
    if (offset) *offset = p.offset;
    if (rows) *rows = p.rows;
    if (cols) *cols = p.cols;
    return PTK_OK;
}

extern "C" int ptk_stage_gemm_timing(ptk_stage* st, int enable, double* total_flops, double* total_ms,
                                     long* launches) {
    if (!st) return ptk::set_error(PTK_ERR_ARG, "null stage");
    return guarded("ptk_stage_gemm_timing", [&] {
        ptk::GemmTiming& t = st->impl->gemm_timing();
        st->impl->collect_timing();
        if (total_flops) *total_flops = t.total_flops;
        if (total_ms) *total_ms = t.total_ms;
        if (launches) *launches = t.launches;
        if (enable >= 0) {
            t.armed = enable != 0;
            t.enabled = t.armed;
            if (t.armed) t.stride = enable > 1 ? enable : 8;  // executor: time one micro-batch in `stride`
            t.total_flops = t.total_ms = 0.0;
            t.launches = 0;
        }
    });
}

extern "C" size_t ptk_stage_stash_bytes(ptk_stage* st) { return st ? st->impl->stash_bytes_per_slot() : 0; }
