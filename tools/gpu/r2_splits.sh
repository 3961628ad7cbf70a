# cfg4 geometry (13 image blocks, 91 one-CTA Gram tiles): pixel splits per tile
mkdir -p gpurun_out
for ns in 8 13 16 24; do echo "splits=$ns"; FKK_GRAM_SPLITS=$ns timeout 600 python tools/prof_cfg4.py 2000000 3 2>&1 | grep -v Warn | tail -1 | cut -c1-80; done
