// vgpu-b200 — the paper's closed-form execution-time model (Eqs. 1-11).
//
// Declarations match proj/include/vgpu/model.hpp:27-56. With A = t_data_in,
// B = t_comp, C = t_data_out and N processes:
//   no virtualization : N (T_init + A + B + C) + (N - 1) T_ctx
//   PS-1              : N (A + C) + B
//   PS-2 (general)    : A + B + C + (N - 1) max(A, B, C)
//   PS-2, C-I         : A + N B + C
//   PS-2, IO-I        : N max(A, C) + B + min(A, C)
// The GVM uses classify_kernel + recommend_style to pick each batch's issue
// order; the totals feed the model-vs-measured report.
#ifndef VGPU_MODEL_HPP
#define VGPU_MODEL_HPP

#include "vgpu/types.hpp"

namespace vgpu {

KernelClass classify_kernel(const KernelProfile& p);
ProgrammingStyle recommend_style(KernelClass c);

Micros t_total_no_vt(const ModelParams& m);
Micros t_total_ci_ps1(const ModelParams& m);
Micros t_total_ci_ps2(const ModelParams& m);
Micros t_total_ioi_ps1(const ModelParams& m);
Micros t_total_ioi_ps2(const ModelParams& m);

Micros t_total_ps1(const ModelParams& m);
Micros t_total_ps2(const ModelParams& m);

struct StyleComparison {
    Micros ps1_total;
    Micros ps2_total;
    ProgrammingStyle preferred;  // ties go to PS1
};
StyleComparison compare_styles(const ModelParams& m);

double speedup_ci(const ModelParams& m);
double speedup_ioi(const ModelParams& m);
double speedup_limit_ci(const ModelParams& m);
double speedup_limit_ioi(const ModelParams& m);

}  // namespace vgpu

#endif  // VGPU_MODEL_HPP
