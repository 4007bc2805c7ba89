# A/B of the attention kernels: working-tree library (B) vs ab/libchunkft_b200_base.so (A),
# alternating three times on one box.
cp paper_2605_21177_b200/_native/libchunkft_b200.so /tmp/lib_b.so
for i in 1 2 3; do
  cp ab/libchunkft_b200_base.so paper_2605_21177_b200/_native/libchunkft_b200.so
  echo "A $(python scripts/attn_probe.py 30 | tr '\n' ' ')"
  cp /tmp/lib_b.so paper_2605_21177_b200/_native/libchunkft_b200.so
  echo "B $(python scripts/attn_probe.py 30 | tr '\n' ' ')"
done
