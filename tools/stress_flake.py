import sys, os
sys.path.insert(0, os.getcwd())
import tests.test_parity_gpu as P
n = 0
for it in range(25):
    for mode in (0, 1):
        P.test_degenerate_shapes_exact(mode)
        P.test_batch_population_exact(mode)
        n += 2
    P.test_cfg1_all_variants_exact(it % 3, True, 1)
print("ok", n)
