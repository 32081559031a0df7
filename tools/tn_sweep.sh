for c in 148 296 444 592; do LRX_GEMM_TN_CTAS=$c timeout 120 python tools/gemm_bench2.py . 2>&1 | sed "s/^/ctas=$c /"; done
LRX_GEMM_TN_MT2=1 LRX_GEMM_TN_CTAS=148 timeout 120 python tools/gemm_bench2.py . | sed "s/^/mt2 148 /"
