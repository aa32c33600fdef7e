// abcq_gemv_lut.cu -- launcher of the sm_100a batch-1 GEMV (kernel: abcq_gemv_lut.cuh).
#include "abcq_gemv_lut.cuh"

namespace abcq {

size_t lut_workspace_bytes(const abcq_model_t* m) {
    const int NRT = n_row_tiles(m->rows), NS = n_slices(m->cols);
    if (NS <= 1) return 0;
    return (size_t)NS * NRT * kTileRows * sizeof(float);
}

bool lut_supports(const abcq_model_t* m, int p) { return m->layout == ABCQ_LAYOUT_TILED && p <= kMaxFastP; }

template <typename XT>
static int launch_yt(const LutArgs& a, int yd, int sd, bool asym, int grid, cudaStream_t st) {
    return yd == ABCQ_F16 ? launch_lut_xy<XT, __half>(a, sd, asym, grid, st)
                          : launch_lut_xy<XT, float>(a, sd, asym, grid, st);
}

unsigned long long* g_trace = nullptr;  // abcq_debug_set_trace (profiling aid)
int g_dbg_mode = 0;                     // abcq_debug_set_mode (profiling experiments)

int launch_gemv_lut(const abcq_model_t* m, int p, const void* x, int x_dtype, void* y, int y_dtype,
                    void* ws, cudaStream_t st) {
    LutArgs a;
    a.rows = m->rows;
    a.cols = m->cols;
    a.NRT = n_row_tiles(m->rows);
    a.NS = n_slices(m->cols);
    a.p = p;
    a.items = a.NRT * a.NS;
    a.planes = static_cast<const uint4*>(m->planes);
    a.plane_stride_u4 = m->plane_stride_bytes / 16;
    a.alpha = m->alpha[p];
    a.offset = m->asymmetric ? m->offset[p] : nullptr;
    // trace ring: 16 launch slots of (kTraceCtas x 8) stamps; the slot is fixed
    // at launch (and capture) time
    static unsigned trace_seq = 0;
    a.trace = g_trace ? g_trace + (size_t)(trace_seq++ % 16) * kTraceCtas * 8 : nullptr;
    a.dbg_mode = g_dbg_mode;
    a.x = x;
    a.y = y;
    a.partial = static_cast<float*>(ws);
    int grid = num_sms();
    if (grid < a.NS) grid = a.NS;      // keeps every CTA within <= 2 slices
    if (grid > a.items) grid = a.items;
    a.q = a.items / grid;
    a.rem = a.items % grid;
    const bool asym = m->asymmetric != 0;
    return x_dtype == ABCQ_F16 ? launch_yt<__half>(a, y_dtype, m->scale_dtype, asym, grid, st)
                               : launch_yt<float>(a, y_dtype, m->scale_dtype, asym, grid, st);
}

}  // namespace abcq
