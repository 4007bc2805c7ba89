# Attention forward vs the share of exponentials computed on the FMA pipe (CFT_POLY_SHARE of 4),
# rebuilt on the box for each share; restores the default build at the end.
for s in 0 1 2 3 4; do
  rm -f paper_2605_21177_b200/_native/obj/attn_fa.o
  make -C paper_2605_21177_b200 -j8 EXTRA_NVFLAGS=-DCFT_POLY_SHARE=$s > /dev/null 2>&1 || echo "build $s failed"
  echo "share $s/4: $(python scripts/attn_probe.py 20 | head -1)"
done
rm -f paper_2605_21177_b200/_native/obj/attn_fa.o
make -C paper_2605_21177_b200 -j8 > /dev/null 2>&1
