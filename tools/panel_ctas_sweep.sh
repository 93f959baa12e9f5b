# he2hb time vs the panel's CTA cap (EIG_PANEL_CTAS), small and large n
for c in 4 8 12 16 24 32; do
  echo "== EIG_PANEL_CTAS=$c"
  for n in 2000 5000 10000; do EIG_PANEL_CTAS=$c timeout 120 python tools/prof_kernels.py he2hb --n $n --m3; done
done
