// precision variant: u storage float, u_f storage float, operator MODE_F64
#include "gb_solver.cuh"

const VariantOps* gb_variant_f_f_f64() { return Impl<float, float, MODE_F64>::table(); }
