S = "[('hval','eval_kernel.cuh',117,138),('prefetch','eval_kernel.cuh',159,266),('bus_terms','eval_kernel.cuh',267,311),('A_end','eval_kernel.cuh',312,439),('gens','eval_kernel.cuh',440,460),('copyfn','eval_kernel.cuh',461,505),('setup','eval_kernel.cuh',506,592),('A','eval_kernel.cuh',593,612),('B','eval_kernel.cuh',613,649),('C','eval_kernel.cuh',650,667)]"
print(S)
