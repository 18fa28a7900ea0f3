#!/bin/bash
# A/B of ab/libA.so vs ab/libB.so on the cfg3 GLA forward / backward (tools/bwd_vec_time.py)
export PYTHONPATH=.
for rep in 1 2 3; do
  for v in A B; do echo "$v $(LMOE_LIB=ab/lib$v.so timeout 120 python tools/bwd_vec_time.py x 262144 gla 2>&1 | tail -2 | tr '\n' ' ')"; done
done
