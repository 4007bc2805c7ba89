# Attention kernels: suspend-hint waits (default) vs polling waits, and the poly share.
for v in "" "-DCFT_ATTN_SPIN" "-DCFT_POLY_SHARE=0" "-DCFT_POLY_SHARE=2"; do
  rm -f paper_2605_21177_b200/_native/obj/attn_fa.o
  make -C paper_2605_21177_b200 -j8 EXTRA_NVFLAGS="$v" > /dev/null 2>&1 || echo "build $v failed"
  echo "[$v] $(python scripts/attn_probe.py 20 | tr '\n' ' ')"
done
rm -f paper_2605_21177_b200/_native/obj/attn_fa.o
make -C paper_2605_21177_b200 -j8 > /dev/null 2>&1
