// precision variant: u storage double, u_f storage float, operator MODE_F64
#include "gb_solver.cuh"

const VariantOps* gb_variant_d_f_f64() { return Impl<double, float, MODE_F64>::table(); }
