# Mutation check of the oracle pins beyond the separator code (scripts/oracle_mutations.sh):
# the network build (R1 split, Thm 2 placement), the pairwise contraction, the bitstring
# and slice handling, the Eq. (3) cost counts and the Theorem 1 closed form.  Each
# mutation is applied to a scratch copy; the CPU oracle tests must FAIL by assertion.
# (Theorem 1's exponent n^{1-1/d} equals n^{1/d} at d = 2, the only dimension of the
# configs, so that swap is unobservable; its constant a_2 = 4 + 2 sqrt(3) is pinned.)
# usage: bash scripts/oracle_mutations_all.sh
set -u
SRC=$(cd "$(dirname "$0")/.." && pwd)
MUTS=(
  "split_transposed|network.py|s/Y\[i, j, k\] = U\[2 \* (k >> 1) + i, 2 \* (k \& 1) + j\]/Y[i, j, k] = U[2 * (k >> 1) + j, 2 * (k \& 1) + i]/"
  "diag_split_swapped|network.py|s/Y\[i, i, k\] = U\[2 \* k + i, 2 \* k + i\]/Y[i, i, k] = U[2 * i + k, 2 * i + k]/"
  "x_half_at_midpoint|network.py|s/pa = (float(xa\[0\] + (xb\[0\] - xa\[0\]) \/ 4.0)/pa = (float(xa[0] + (xb[0] - xa[0]) \/ 2.0)/"
  "input_state_one|network.py|s/add(\[wire\[q\]\], \[1.0, 0.0\]/add([wire[q]], [0.0, 1.0]/"
  "matmul_conjugated|contract.py|s/C = np.matmul(A2, B2)/C = np.matmul(A2.conj(), B2)/"
  "bitstring_flipped|contract.py|s/fix\[net.out_leg\[q\]\] = int(bits\[q\])/fix[net.out_leg[q]] = 1 - int(bits[q])/"
  "slices_not_summed|contract.py|s/        total += r/        total = r/"
  "cost_counts_kept_only|ssa.py|s/out.append((sum(l2\[i\] for i in union), /out.append((sum(l2[i] for i in kept), /"
  "sliced_work_no_multiplicity|ssa.py|s/return w \* 2.0 \*\* sum(l2\[i\] for i in sl)/return w/"
  "thm1_constant|bounds.py|s/return C_D\[d\] \/ (2.0 - 2.0/return C_D[d] \/ (2.0 - 1.0/"
)
rc_all=0
for m in "${MUTS[@]}"; do
  IFS='|' read -r name file expr <<< "$m"
  D=$(mktemp -d)
  cp -r "$SRC/oracle" "$SRC/tests" "$SRC/tn_inputs" "$D/"
  sed -i "$expr" "$D/oracle/$file"
  if cmp -s "$SRC/oracle/$file" "$D/oracle/$file"; then echo "$name: MUTATION NOT APPLIED"; rc_all=1; rm -rf "$D"; continue; fi
  (cd "$D" && timeout 900 python -m pytest tests/test_oracle_ssa_pins.py tests/test_oracle.py -x -q -m "not gpu" -p no:cacheprovider > out.txt 2>&1)
  rc=$?
  if [ $rc -eq 1 ]; then echo "$name: caught ($(grep -m1 -E '^FAILED' "$D/out.txt" | cut -c1-110))"
  else echo "$name: NOT CAUGHT (pytest rc=$rc)"; rc_all=1; fi
  rm -rf "$D"
done
exit $rc_all
