# Mutation check of the oracle pins: apply each mutation to a scratch copy of the repo
# and run the CPU oracle tests; every mutation must FAIL by assertion (not by timeout).
# usage: bash scripts/oracle_mutations.sh
set -u
SRC=$(cd "$(dirname "$0")/.." && pwd)
declare -A MUT
MUT[classify_radius_x2]='s/^def classify(sep, PX, PY, rad):/def classify(sep, PX, PY, rad):\n    rad = 2.0 * rad/'
MUT[eq2_loosened_7_8]='s/if 4 \* nE > 3 \* s or 4 \* nI > 3 \* s:/if 8 * nE > 7 * s or 8 * nI > 7 * s:/'
MUT[greedy_max_cost]='s/key = (cost, res, min(A.nid, B.nid), max(A.nid, B.nid))/key = (-cost, res, min(A.nid, B.nid), max(A.nid, B.nid))/'
MUT[boundary_inverted]='s/        if wE > wI:/        if wE < wI:/; s/        elif wI > wE:/        elif wI < wE:/'
MUT[eq1_dropped]='s/if not float(nO \* nO) <= (C_D\[2\] \* C_D\[2\]) \* k \* float(s):/if False:/'
MUT[selection_max_cut]='s/if best is None or cut < best\[2\]:/if best is None or cut > best[2]:/'
MUT[median_narrow_axis]='s/key = PX if wx >= wy else PY/key = PY if wx >= wy else PX/'
MUT[tie_rule_flipped]='s/side = 1 if len(E) <= len(I) else 2/side = 2 if len(E) <= len(I) else 1/'
rc_all=0
for name in "${!MUT[@]}"; do
  D=$(mktemp -d)
  cp -r "$SRC/oracle" "$SRC/tests" "$SRC/tn_inputs" "$D/"
  sed -i "${MUT[$name]}" "$D/oracle/ssa.py"
  if cmp -s "$SRC/oracle/ssa.py" "$D/oracle/ssa.py"; then echo "$name: MUTATION NOT APPLIED"; rc_all=1; continue; fi
  (cd "$D" && timeout 900 python -m pytest tests/test_oracle_ssa_pins.py tests/test_oracle.py -x -q -m "not gpu" -p no:cacheprovider > out.txt 2>&1)
  rc=$?
  if [ $rc -eq 1 ]; then echo "$name: caught ($(grep -m1 -E '^FAILED' "$D/out.txt" | cut -c1-110))"
  else echo "$name: NOT CAUGHT (pytest rc=$rc)"; rc_all=1; fi
  rm -rf "$D"
done
exit $rc_all
