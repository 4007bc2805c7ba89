# Attention forward vs CFT_POLY_SHARE (exponentials per 4 on the FMA pipe), rebuilt on the box.
for v in 0 1 2; do
  rm -f paper_2605_21177_b200/_native/obj/attn_fa.o
  make -C paper_2605_21177_b200 -j8 EXTRA_NVFLAGS="-DCFT_POLY_SHARE=$v" > /dev/null 2>&1 || echo "build $v failed"
  echo "share $v: $(python scripts/attn_probe.py 30 | tr '\n' ' ')"
done
rm -f paper_2605_21177_b200/_native/obj/attn_fa.o
make -C paper_2605_21177_b200 -j8 > /dev/null 2>&1
