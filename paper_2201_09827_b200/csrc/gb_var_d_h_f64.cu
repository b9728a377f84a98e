// precision variant: u storage double, u_f storage __half, operator MODE_F64
#include "gb_solver.cuh"

const VariantOps* gb_variant_d_h_f64() { return Impl<double, __half, MODE_F64>::table(); }
