S = "[('hval','eval_kernel.cuh',117,140),('gath_end','eval_kernel.cuh',166,218),('gath_bus','eval_kernel.cuh',221,262),('A_end','eval_kernel.cuh',263,375),('copyfn','eval_kernel.cuh',376,408),('setup','eval_kernel.cuh',409,489),('A','eval_kernel.cuh',490,509),('B','eval_kernel.cuh',510,545),('sums','eval_kernel.cuh',546,564),('C','eval_kernel.cuh',565,582)]"
print(S)
