#!/bin/bash
tools/ab_session.sh r01b u1 u2 u1_r96 u2_r96 u1_r80 u2_r80
tools/gpu_session.sh r01b tests
