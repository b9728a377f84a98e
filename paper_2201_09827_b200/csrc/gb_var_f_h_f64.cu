// precision variant: u storage float, u_f storage __half, operator MODE_F64
#include "gb_solver.cuh"

const VariantOps* gb_variant_f_h_f64() { return Impl<float, __half, MODE_F64>::table(); }
