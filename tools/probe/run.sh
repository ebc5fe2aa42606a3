#!/bin/bash
cd tools/probe
for b in tma_probe_nohint tma_probe; do for ax in 2 1 0; do echo "== $b axis $ax"; timeout 60 ./$b 36 $ax; done; done
