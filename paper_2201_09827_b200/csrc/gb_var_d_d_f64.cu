// precision variant: u storage double, u_f storage double, operator MODE_F64
#include "gb_solver.cuh"

const VariantOps* gb_variant_d_d_f64() { return Impl<double, double, MODE_F64>::table(); }
