// Opaque handle types of the C ABI.
#pragma once

#include "gpt_stage.h"

struct ptk_stage {
    ptk::GptStage* impl;
    bool owned;
    ptk_stage(ptk::GptStage* p, bool own) : impl(p), owned(own) {}
    ~ptk_stage() {
        if (owned) delete impl;
    }
    ptk_stage(const ptk_stage&) = delete;
    ptk_stage& operator=(const ptk_stage&) = delete;
};
