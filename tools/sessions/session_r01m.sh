#!/bin/bash
tools/ab_session.sh r01m u1 norecip u1 norecip
