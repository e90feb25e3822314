#!/bin/bash
# Strict (1x tolerance) parity fuzz on one B200: contract domain, large frames, stress domain.
O=gpurun_out/${TAG:-fuzz}
mkdir -p $O
S=${SECS:-300}
timeout $((S+120)) python tools/fuzz_parity.py --domain contract --seconds $S --seed ${SEED:-11} --out $O/fail > $O/contract.log 2>&1; echo "rc=$?" >> $O/contract.log
timeout $((S+300)) python tools/fuzz_parity.py --domain contract --large --seconds $S --seed $((${SEED:-11}+1)) --out $O/fail > $O/large.log 2>&1; echo "rc=$?" >> $O/large.log
timeout $((S+120)) python tools/fuzz_parity.py --domain stress --seconds $S --seed $((${SEED:-11}+2)) --out $O/fail > $O/stress.log 2>&1; echo "rc=$?" >> $O/stress.log
for f in $O/*.log; do tail -n 2 $f; done
