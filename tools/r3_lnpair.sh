# LongNet two-tile-per-CTA variant (tools/variants/longnet_umma_pair.cu): trace one CTA, bench cfg4
cp tools/variants/longnet_umma_pair.cu paper_2502_01659_b200/csrc/longnet_umma.cu
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 150 python tools/ln_tiny.py 65536 || { echo "LongNet tiny case failed/hung"; exit 1; }
python tools/build_variant.py ltrace "-DGA_LNET_TRACE" longnet_umma.cu > /dev/null 2>&1
LT_LOADER=8 LT_MMA=9 timeout 300 python tools/lnet_trace.py > gpurun_out/lnpair_trace.txt 2>&1; echo "trace rc=$?"
head -60 gpurun_out/lnpair_trace.txt
