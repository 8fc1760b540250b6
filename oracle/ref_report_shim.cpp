// ref_report_shim.cpp -- C entry point over the UNMODIFIED reference report writer (test
// infrastructure only). Compiled with /root/reference/proj/src/{tensor,rope,collectives,
// kv_cache,sp_attention,generator,report}.cpp into oracle/_ref/libspattn_ref_report.so by
// oracle/Makefile (report.cpp needs nlohmann/json.hpp, which the reference's CMake fetches; a
// copy ships inside the image's cudnn_frontend headers). Nothing here re-implements reference
// logic: it runs spattn::generate and returns to_json(GenerationResult) (report.cpp:161-175)
// with strip_timing_fields (report.cpp:246-262) applied, dumped with indent 2 as cli.cpp does.
#include <cstdint>
#include <cstring>
#include <string>

#include "spattn/generator.hpp"
#include "spattn/report.hpp"

using namespace spattn;

extern "C" {

// cfg as ref_generate (ref_shim.cpp). out: a buffer of cap bytes receiving the JSON text
// (NUL-terminated); *len = its length. Returns 0, 6 if cap is too small, or 1 on a throw.
int ref_report_json(const int64_t* cfg, uint64_t seed, char* out, int64_t cap, int64_t* len) {
    try {
        GenerationConfig c;
        c.grid_per_block = GridSpec{cfg[0], cfg[1], cfg[2]};
        c.num_blocks = cfg[3];
        c.layers = cfg[4];
        c.denoise_steps = cfg[5];
        c.heads = cfg[6];
        c.head_dim = cfg[7];
        c.world_size = static_cast<int>(cfg[8]);
        if (cfg[9] >= 0) c.window_frames = cfg[9];
        const int64_t mask = cfg[11];
        AblationFlags f{(mask & 1) != 0, (mask & 2) != 0, (mask & 4) != 0};
        if (cfg[10] == 0) c.variant = PipelineVariant::reference();
        if (cfg[10] == 1) c.variant = PipelineVariant::baseline();
        if (cfg[10] == 2) c.variant = PipelineVariant::optimized(f);
        c.force_start_frame_zero = cfg[12] != 0;
        c.seed = seed;
        Json j = to_json(generate(c));
        strip_timing_fields(j);
        const std::string s = j.dump(2);
        *len = static_cast<int64_t>(s.size());
        if (static_cast<int64_t>(s.size()) + 1 > cap) return 6;
        std::memcpy(out, s.c_str(), s.size() + 1);
        return 0;
    } catch (...) {
        return 1;
    }
}

}  // extern "C"
