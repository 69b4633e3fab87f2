# A/B of skinny PTDF variants (measurement only)
for v in default paper_2406_13191_b200/lib/variants/*.so; do
  if [ "$v" = default ]; then o=$(python tools/ptdf_gap_explore.py 3 2>&1 | sed -n 3p); else o=$(DCOPF_LIB=$v python tools/ptdf_gap_explore.py 3 2>&1 | sed -n 3p); fi
  echo "$(basename $v) :: $o" | cut -c1-80
done
