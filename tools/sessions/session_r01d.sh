#!/bin/bash
tools/ab_session.sh r01d u1 u1_imm u2
tools/gpu_session.sh r01d ncu
