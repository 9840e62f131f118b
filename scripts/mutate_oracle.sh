#!/usr/bin/env bash
# Mutation check of the oracle pins: apply plausible mistakes to
# oracle/ffn_oracle.c one at a time and require tests/test_oracle.py to fail.
# Restores the source afterwards.  CPU only.
set -u
cd "$(dirname "$0")/.."
SRC=oracle/ffn_oracle.c
cp "$SRC" /tmp/ffn_oracle.orig.c
trap 'cp /tmp/ffn_oracle.orig.c "$SRC"; python -c "import oracle; oracle.build(force=True)"' EXIT
status=0
while IFS= read -r mut; do
  [ -z "$mut" ] && continue
  cp /tmp/ffn_oracle.orig.c "$SRC"; sed -i "$mut" "$SRC"
  if cmp -s /tmp/ffn_oracle.orig.c "$SRC"; then echo "NOT APPLIED: $mut"; status=1; continue; fi
  if timeout 300 python -m pytest tests/test_oracle.py -q >/dev/null 2>&1; then
    echo "SURVIVED: $mut"; status=1
  else
    echo "killed:   $mut"
  fi
done <<'MUTS'
s|r = 1.0 / sqrt(ss / (double)K + eps);|r = 1.0 / (sqrt(ss / (double)K) + eps);|
s|double r = 1.0 / sqrt(ss / (double)K + eps);|double r = 1.0 / sqrt(ss / (double)(K-1) + eps);|
s|double r = 1.0 / sqrt(ss / (double)K + eps);|double r = 1.0 / sqrt(ss + eps);|
s|XN\[i \* K + k\] = (mode == ORACLE_PLAIN) ? v \* r \* G\[k\] : v;|XN[i * K + k] = (mode == ORACLE_PLAIN) ? v * r : v;|
s|out\[i \* N + n0 + j\] = h1 / (1.0 + exp(-h1)) \* h3;|out[i * N + n0 + j] = h3 / (1.0 + exp(-h3)) * h1;|
s|out\[i \* N + n0 + j\] = h1 / (1.0 + exp(-h1)) \* h3;|out[i * N + n0 + j] = h1 / (1.0 + exp(h1)) * h3;|
s|out\[i \* N + n0 + j\] = h1 / (1.0 + exp(-h1)) \* h3;|out[i * N + n0 + j] = 1.0 / (1.0 + exp(-h1)) * h3;|
s|const double\* a = W1 + j \* K;|const double* a = W1 + (j % 2) * K;|
s|a = oracle_round_bf16(a \* G\[k\]);|a = a * G[k];|
s|uint32_t bias = (1u << (drop - 1)) - 1u + lsb;|uint32_t bias = (1u << (drop - 1));|
s|if (mode != ORACLE_PLAIN) { h1 \*= R\[i\]; h3 \*= R\[i\]; }|if (mode != ORACLE_PLAIN) { h1 *= R[i]; }|
s|dst_bits\[n \* K + k\] = oracle_round_bf16_bits(bf16_bits_to_double(w\[n \* K + k\]) \*|dst_bits[n * K + k] = oracle_round_bf16_bits(bf16_bits_to_double(w[n * K + k]) + 0 *|
s|out\[m \* N + n\] = (act == 1 \&\& acc < 0.0) ? alpha \* acc : acc;|out[m * N + n] = (act == 1 \&\& acc < 0.0) ? 0.01 * acc : acc;|
s|acc += load_elem(x, x_dtype, m \* K + k) \* load_elem(w, w_dtype, n \* K + k);|acc += load_elem(x, x_dtype, m * K + k) * load_elem(w, w_dtype, k * N + n % K);|
s|for (int64_t n = 0; n < N; ++n) acc += hid\[i \* N + n\] \* load_elem(w2, w_dtype, j \* N + n);|for (int64_t n = 0; n < N; ++n) acc += hid[i * N + n] * load_elem(w2, w_dtype, n * K + j % N);|
s|for (int64_t i = 0; i < nrows \* N; ++i) hid\[i\] = oracle_round_bf16(hid\[i\]);|for (int64_t i = 0; i < nrows * N; ++i) hid[i] = (double)(float)hid[i];|
s|out\[m \* K + k\] = load_elem(x, x_dtype, m \* K + k) \* r \* load_elem(g, g_dtype, k);|out[m * K + k] = load_elem(x, x_dtype, m * K + k) * r;|
s|a = oracle_round_tf32((double)(float)(a \* G\[k\]));|a = a * G[k];|
s|b = oracle_round_tf32((double)(float)(b \* G\[k\]));|b = oracle_round_bf16(b * G[k]);|
MUTS
exit $status
