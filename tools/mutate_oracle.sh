#!/bin/bash
# Mutation check of the oracle pins: each mutation of oracle/oracle.c must make
# tests/test_oracle_pins.py fail.  Restores the source and rebuilds at the end.
cd "$(dirname "$0")/.."
cp oracle/oracle.c /tmp/oracle.c.orig
trap 'cp /tmp/oracle.c.orig oracle/oracle.c; python -c "import oracle; oracle.build(force=True)"' EXIT
muts=(
 's/reallocate(h, (long)mv + k_adm, mv);/reallocate(h, (long)mv + k_adm + 5, mv);/'
 's/reallocate(h, (long)mv + k_adm, mv);/reallocate(h, (long)mv + k_adm, mv > 0 ? mv - 1 : 0);/'
 's/int rc = reallocate(h, (long)mv + 1, mv);/int rc = reallocate(h, (long)mv + 2, mv);/'
 's/h->st.kv_bytes_read += 2LL \* units(h) \* h->cap/h->st.kv_bytes_read += 2LL * units(h) * (h->cap - h->staged)/'
 's/long nc = h->cap + h->r;/long nc = h->cap + h->r + 1;/'
 's/int rc = reallocate(h, nc, h->cap);/int rc = reallocate(h, nc, h->cap - 1);/'
 's/if (!h->tree) return j < vb + tau;/if (!h->tree) return j <= vb + tau;/'
 's/const double scale = 1.0 \/ sqrt((double)h->D);/const double scale = 1.0 \/ (double)h->D;/'
 's/for (int i = m; i < h->staged; ++i) {/for (int i = m + 1; i < h->staged; ++i) {/'
 's/int k_adm = (long)k < free_rows ? k : (int)free_rows;/int k_adm = k;/'
 's/long u = (long)b \* h->H_kv + hq \/ G;/long u = (long)b * h->H_kv + hq % h->H_kv;/'
)
fail=0
for m in "${muts[@]}"; do
  cp /tmp/oracle.c.orig oracle/oracle.c; sed -i "$m" oracle/oracle.c
  if cmp -s oracle/oracle.c /tmp/oracle.c.orig; then echo "NOT APPLIED  $m"; fail=1; continue; fi
  python -c "import oracle; oracle.build(force=True)"
  if timeout 900 python -m pytest tests/test_oracle_pins.py -q -x -p no:cacheprovider >/dev/null 2>&1; then
    echo "SURVIVED     $m"; fail=1
  else
    echo "caught       $m"
  fi
done
exit $fail
