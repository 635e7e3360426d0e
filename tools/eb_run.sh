# kappa scan of the round-toward-zero compensation (tools/error_budget.py), forward drain 1
for k in 2.5e-8 3.0e-8 3.5e-8 4.0e-8; do
  SPST_RZ_KAPPA=$k python tools/error_budget.py --out gpurun_out/eb_k$k.json > gpurun_out/eb_k$k.log 2>&1
done
SPST_RZ_KAPPA=0 python tools/error_budget.py --points 0 --out gpurun_out/eb_k0.json > gpurun_out/eb_k0.log 2>&1
