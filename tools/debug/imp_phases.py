import bench
r = bench.implicit_measure(0, cpu=False)
print({k: r[k] for k in ("ms_per_be_step", "cg_per_step", "us_per_cg_iteration", "pcg_solve")})
