// precision variant: u storage float, u_f storage __half, operator MODE_F32
#include "gb_solver.cuh"

const VariantOps* gb_variant_f_h_f32() { return Impl<float, __half, MODE_F32>::table(); }
