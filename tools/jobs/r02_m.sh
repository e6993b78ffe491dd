#!/bin/bash
# Parareal behaviour: coarse-propagator damping (theta_c = 1/2 + theta0 K, 25 -> implicit Euler at K = 0.02),
# temporal order with pure CN / short horizon, c2 with a damped coarse propagator
mkdir -p gpurun_out
A="timeout 900 python tools/parareal_analysis.py"
$A fields --config c1 --variants classic --coarse-theta0 25 > gpurun_out/m_fields.jsonl 2> gpurun_out/m_fields.err
$A fields --config c1 --variants classic --coarse-theta0 5 >> gpurun_out/m_fields.jsonl 2>> gpurun_out/m_fields.err
$A fields --config c1 --variants classic --coarse-theta0 25 --iters 10 >> gpurun_out/m_fields.jsonl 2>> gpurun_out/m_fields.err
$A fields --config c2 --variants classic --coarse-theta0 25 >> gpurun_out/m_fields.jsonl 2>> gpurun_out/m_fields.err
$A fields --config c2 --variants classic >> gpurun_out/m_fields.jsonl 2>> gpurun_out/m_fields.err
$A order --config c1 --theta0 0 > gpurun_out/m_order.jsonl 2> gpurun_out/m_order.err
$A order --config c1 --t-final 0.05 --steps 0.002 0.001 0.0005 0.00025 >> gpurun_out/m_order.jsonl 2>> gpurun_out/m_order.err
true
